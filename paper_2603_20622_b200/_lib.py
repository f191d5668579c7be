"""ctypes binding of librtec.so (the C ABI declared in include/rtec.h).

The library is built in-tree (`paper_2603_20622_b200/librtec.so`, see
`__graft_entry__.build()`).  There is no fallback: if the library or a CUDA
device is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtec.so")

OP_INSERT = 0
OP_DELETE = 1
MODEL_IDS = {"gcn": 0, "graphsage": 1, "gin": 2, "gat": 3, "gin_max": 4, "pinsage": 5, "monet": 6, "commnet": 7,
             "ggcn": 8, "agnn": 9}
ARENA_FULL = 8
ERR_OK = (1 << 64) - 1

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
SZ = C.c_size_t
F32 = C.c_float


class Adj(C.Structure):
    _fields_ = [("slots", I64), ("beg", P), ("len", P), ("cap", P), ("nbr", P), ("ts", P), ("top", P)]


class Graph(C.Structure):
    _fields_ = [
        ("n", I64), ("out", Adj), ("inn", Adj),
        ("out_deg", P), ("in_deg", P), ("out_deg_prev", P), ("in_deg_prev", P),
        ("num_edges", P), ("slack", F32), ("min_slack", I32), ("part_rank", I32), ("part_count", I32),
    ]


class Batch(C.Structure):
    _fields_ = [
        ("cap", I64), ("err", P), ("status", P),
        ("a_src", P), ("a_dst", P), ("a_op", P), ("a_ts", P), ("n_applied", P),
        ("i_src", P), ("i_dst", P), ("i_op", P),
        ("d_vertex", P), ("d_old_in", P), ("d_new_in", P), ("d_old_out", P), ("d_new_out", P),
        ("n_delta", P), ("irange", P), ("dg_bm", P), ("apply_ctr", P),
    ]


class Frontier(C.Structure):
    _fields_ = [
        ("bm_src", P), ("bm_dst", P), ("src_list", P), ("n_src", P), ("dst_list", P), ("n_dst", P),
        ("src_slot", P), ("dst_slot", P), ("counters", P), ("bm_chg", P), ("chg_slot", P),
    ]


class Layer(C.Structure):
    _fields_ = [
        ("model", I32), ("d_in", I32), ("d_out", I32), ("heads", I32),
        ("degree_offset", F32), ("pad", I32), ("W", P), ("W2", P), ("att", P),
        ("Wt_hi", P), ("Wt_lo", P), ("W2t_hi", P), ("W2t_lo", P), ("Wp", P), ("bp", P), ("scalar", F32),
        ("d_k", I32),
    ]


class State(C.Structure):
    _fields_ = [
        ("H_in", P), ("H_out", P), ("S", P), ("ctx", P), ("log_out", P), ("log_in", P),
        ("Z", P), ("el", P), ("er", P), ("Z_log", P), ("er_log", P), ("gemm_in", P), ("gemm_mid", P),
        ("delta", P), ("delta_next", P), ("delta_ready", I32), ("row_div", I32), ("out_local", I32),
        ("delta_slot", I32),
    ]


class Shard(C.Structure):
    _fields_ = [
        ("rank", I32), ("world", I32), ("n", I64), ("n_own", I64), ("cap", I64), ("g2l", P), ("l2g", P),
        ("n_loc", P), ("peers", P), ("gout", P), ("gout_prev", P),
    ]


_SIGS = {
    "rtec_workspace_bytes": (SZ, [I64, I64, I64, I32]),
    "rtec_workspace_bytes_ext": (SZ, [I64, I64, I64, I32]),
    "rtec_build_workspace_bytes": (SZ, [I64, I64]),
    "rtec_graph_count": (C.c_int, [P, P, I64, I64, P, P, P, P]),
    "rtec_graph_slots_needed": (C.c_int, [P, I64, F32, I32, P, P, SZ, P]),
    "rtec_graph_build": (C.c_int, [C.POINTER(Graph), P, P, P, I64, F32, I32, P, P, SZ, P]),
    "rtec_adj_compact": (C.c_int, [I64, C.POINTER(Adj), C.POINTER(Adj), F32, I32, P, SZ, P]),
    "rtec_adj_export": (C.c_int, [I64, C.POINTER(Adj), P, P, P, P, SZ, P]),
    "rtec_batch_coalesce": (C.c_int, [P, P, P, P, I64, P, P, P, P, P, P, SZ, P]),
    "rtec_batch_apply": (C.c_int, [C.POINTER(Graph), C.POINTER(Batch), P, P, P, P, I64, P, SZ, P]),
    "rtec_batch_apply_phase": (C.c_int, [C.POINTER(Graph), C.POINTER(Batch), P, P, P, P, I64, I32, P, SZ, P]),
    "rtec_batch_commit": (C.c_int, [C.POINTER(Graph), C.POINTER(Batch), P]),
    "rtec_batch_validate": (C.c_int, [P, P, I64, I64, P, P, SZ, P]),
    "rtec_shard_admit": (C.c_int, [C.POINTER(Shard), P, P, P, I64, P, P, P, P, P, P, P, P, P, SZ, P]),
    "rtec_shard_localize": (C.c_int, [C.POINTER(Shard), P, P, P, P, I64, P, P, P, P, P, P, P, P, SZ, P]),
    "rtec_shard_count_peers": (C.c_int, [C.POINTER(Shard), P, P, I64, P, P]),
    "rtec_shard_pack": (C.c_int, [C.POINTER(Shard), I32, P, P, P, P, P, I64, P, P, I64, P, P, P, P, P]),
    "rtec_shard_unpack_rows": (C.c_int, [C.POINTER(Shard), I32, P, P, P, P, P, I64, P, P]),
    "rtec_shard_unpack_changed": (C.c_int, [C.POINTER(Shard), I32, P, P, I64, I64, I32, P, P, P, I64, P, P, P, P,
                                            I32, F32, P, P, P, P, P]),
    "rtec_shard_degrees": (C.c_int, [C.POINTER(Shard), P, P, P, P, I64, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "rtec_shard_commit": (C.c_int, [C.POINTER(Shard), P, P, P, I64, P, P, P]),
    "rtec_frontier_layer": (C.c_int, [C.POINTER(Graph), C.POINTER(Batch), I32, I32, C.POINTER(Frontier),
                                      C.POINTER(Frontier), P, SZ, P]),
    "rtec_layer_incremental": (C.c_int, [C.POINTER(Graph), C.POINTER(Batch), C.POINTER(Layer), C.POINTER(State),
                                         C.POINTER(Frontier), C.POINTER(Frontier), P, P, SZ, P]),
    "rtec_layer_full": (C.c_int, [C.POINTER(Graph), C.POINTER(Layer), C.POINTER(State), P, P, I64, P, P, SZ, P]),
    "rtec_gat_project": (C.c_int, [C.POINTER(Layer), P, P, P, I64, P, P, P, P, P, P, P, P]),
    "rtec_project": (C.c_int, [C.POINTER(Layer), P, P, P, I64, P, P, P, P]),
    "rtec_update_gemm": (C.c_int, [P, I64, P, I32, I32, P, I64, I32, P, I64, P, P, P, P]),
    "rtec_query": (C.c_int, [P, I64, P, I64, P, I32, P, P]),
    "rtec_ns_sample": (C.c_int, [C.POINTER(Adj), P, P, I64, I32, C.c_uint64, I32, C.POINTER(Adj), P, I64, P, SZ, P]),
    "rtec_bitmap_to_list": (C.c_int, [P, I64, P, P, P, SZ, P]),
    "rtec_in_expand": (C.c_int, [C.POINTER(Adj), P, P, I64, P, P]),
    "rtec_gemm_prepare_weights": (C.c_int, [P, I32, I32, P, P, P]),
    "rtec_struct_sizes": (None, [C.POINTER(I64)]),
    "rtec_prof_enable": (None, [C.c_int]),
    "rtec_prof_report": (SZ, [C.c_char_p, SZ, C.c_int]),
    "rtec_last_error": (C.c_char_p, []),
    "rtec_graph_kernel_nodes": (I64, [P]),
    "rtec_version": (C.c_char_p, []),
    "rtec_device_sm_count": (C.c_int, []),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(require_cuda: bool = True):
    """Load librtec.so; raises NativeError if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise E.NativeError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise E.NativeError("librtec needs a CUDA device (B200); none is visible")
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (_lib.rtec_last_error() or b"").decode(errors="replace")
    cls = E.BY_CODE.get(status)
    if cls is None:
        raise E.NativeError(f"{what}: status {status}: {msg}")
    raise cls(f"{what}: {msg}")


def decode_err(word: int):
    """Device status word -> (code, position) or None when ok."""
    word = int(word) & ERR_OK
    if word == ERR_OK:
        return None
    return word & 0xFFFFFFFF, word >> 32


def raise_err(word: int, what: str, messages=None) -> None:
    d = decode_err(word)
    if d is None:
        return
    code, pos = d
    cls = E.BY_CODE.get(code)
    text = (messages or {}).get(code, f"status {code} at position {pos}")
    if cls is None:
        raise E.NativeError(f"{what}: {text}")
    raise cls(f"{what}: {text}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle():
    import torch

    return torch.cuda.current_stream().cuda_stream


_prof_on = False


def prof_enable(on: bool) -> None:
    """Toggle the library's per-kernel CUDA-event hook (bench / profiling only)."""
    global _prof_on
    _prof_on = bool(on)
    load().rtec_prof_enable(1 if on else 0)


def prof_enabled() -> bool:
    return _prof_on


def prof_report(reset: bool = True) -> dict:
    """Per-kernel {name: (launches, total_ms)} from the library's event hook."""
    n = _lib.rtec_prof_report(None, 0, 0)
    buf = C.create_string_buffer(n + 1)
    _lib.rtec_prof_report(buf, n + 1, 1 if reset else 0)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out
