"""GPU-resident dynamic graph with the reference's DynamicGraph API.

Mirrors `streamgnn/graph.py` (graph.py:28-266): `UpdateOp`, `EdgeUpdate`,
`DegreeDelta`, `ApplyResult`, `DynamicGraph` (from_edges, apply_batch,
in/out neighbours, degrees, has_edge, edges, copy), `coalesce_batch` and
`invert_batch`.  Storage is two gapped adjacencies in HBM (out runs with
timestamps, in runs) maintained by librtec (`graph.cu`); every query and
mutation goes through the C ABI.  Returned numpy arrays are host copies owned
by the caller.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _lib
from . import errors as E

_MAX_KEY = 1 << 62  # pma.MAX_KEY: composite keys src*n+dst stay below it


class UpdateOp(enum.Enum):  # graph.py:28-30
    INSERT = "+"
    DELETE = "-"


@dataclass(frozen=True, slots=True)
class EdgeUpdate:  # graph.py:33-38
    op: UpdateOp
    src: int
    dst: int
    ts: int = 0


@dataclass(frozen=True, slots=True)
class DegreeDelta:  # graph.py:41-48
    vertex: int
    old_in: int
    new_in: int
    old_out: int
    new_out: int


@dataclass(frozen=True, slots=True)
class ApplyResult:  # graph.py:52-56
    applied: tuple
    rejected: tuple
    deltas: tuple


def _device(device=None) -> torch.device:
    _lib.load()
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def updates_to_arrays(batch: Sequence[EdgeUpdate]):
    """Object list -> (op u8, src, dst, ts) int arrays (op 0 = '+', 1 = '-')."""
    B = len(batch)
    op = np.fromiter((0 if u.op is UpdateOp.INSERT else 1 for u in batch), np.uint8, B)
    src = np.fromiter((u.src for u in batch), np.int64, B)
    dst = np.fromiter((u.dst for u in batch), np.int64, B)
    ts = np.fromiter((u.ts for u in batch), np.int64, B)
    return op, src, dst, ts


def _i32_ids(a: np.ndarray) -> np.ndarray:
    """Clamp ids into int32 for the device while preserving 'out of range'."""
    a = np.asarray(a, np.int64)
    return np.where((a < -(1 << 31)) | (a >= (1 << 31)), -1, a).astype(np.int32)


class _Adj:
    """One direction of the adjacency (rtec_adj_t) as torch tensors."""

    def __init__(self, n: int, slots: int, dev, with_ts: bool):
        self.beg = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        self.len = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.cap = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.nbr = torch.empty(max(slots, 1), dtype=torch.int32, device=dev)
        self.ts = torch.empty(max(slots, 1), dtype=torch.int64, device=dev) if with_ts else None
        self.top = torch.zeros(1, dtype=torch.int64, device=dev)
        self.slots = slots

    def c(self) -> _lib.Adj:
        p = _lib.ptr
        return _lib.Adj(self.slots, p(self.beg), p(self.len), p(self.cap), p(self.nbr), p(self.ts), p(self.top))


class DeviceBatch:
    """rtec_batch_t buffers (capacity `cap` updates)."""

    def __init__(self, cap: int, dev, n: int):
        cap = max(int(cap), 1)
        self.cap = cap
        # per-vertex (first, count) into the in-key list, (-1, 0) when untouched
        self.irange = torch.stack([torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev),
                                   torch.zeros(max(n, 1), dtype=torch.int32, device=dev)], dim=1).contiguous()
        z = lambda k, dt: torch.zeros(k, dtype=dt, device=dev)  # noqa: E731
        self.err = z(1, torch.int64)
        self.status = z(cap, torch.uint8)
        self.a_src, self.a_dst, self.a_op, self.a_ts = z(cap, torch.int32), z(cap, torch.int32), z(cap, torch.uint8), z(cap, torch.int64)
        self.n_applied = z(1, torch.int64)
        self.i_src, self.i_dst, self.i_op = z(cap, torch.int32), z(cap, torch.int32), z(cap, torch.uint8)
        self.d = [z(2 * cap, torch.int32) for _ in range(5)]
        self.n_delta = z(1, torch.int64)
        self.apply_ctr = z(4, torch.int64)  # run-merge volume of the last apply (rtec_batch_t.apply_ctr)
        # staging of the batch itself
        self.src, self.dst = z(cap, torch.int32), z(cap, torch.int32)
        self.op, self.ts = z(cap, torch.uint8), z(cap, torch.int64)

    def c(self) -> _lib.Batch:
        p = _lib.ptr
        d = self.d
        return _lib.Batch(self.cap, p(self.err), p(self.status), p(self.a_src), p(self.a_dst), p(self.a_op),
                          p(self.a_ts), p(self.n_applied), p(self.i_src), p(self.i_dst), p(self.i_op),
                          p(d[0]), p(d[1]), p(d[2]), p(d[3]), p(d[4]), p(self.n_delta), p(self.irange), None,
                          p(self.apply_ctr))


class DynamicGraph:
    """Directed graph over [0, n) in B200 HBM (graph.py:59-235 semantics)."""

    # device buffers a captured CUDA graph bakes in: rebinding any of them (compaction, a larger
    # batch or workspace) bumps `layout_version`, the engine's graph-cache key
    _LAYOUT_ATTRS = frozenset({"ws", "batch", "out", "inn", "out_deg", "in_deg", "out_deg_prev", "in_deg_prev",
                               "num_edges_t"})

    def __setattr__(self, name, value):
        if name in DynamicGraph._LAYOUT_ATTRS:
            object.__setattr__(self, "layout_version", self.__dict__.get("layout_version", 0) + 1)
        object.__setattr__(self, name, value)

    def __init__(self, num_vertices: int, *, segment_slots: int = 64,
                 density_bounds: tuple[float, float] = (0.25, 0.875), device=None, slack: float | None = None,
                 min_slack: int = 4, reserve: int | None = None):
        """`segment_slots` / `density_bounds` are the reference's PMA knobs (graph.py:62-68,
        pma.py:40-57), validated with the same rules.  Here every vertex run is its own
        gapped segment: a run of length k gets max(min_slack, ceil(slack * k)) free slots,
        and `slack` defaults to the free fraction the upper density bound leaves
        (1/hi - 1, at least 0.25)."""
        n = int(num_vertices)
        if n < 0 or n * n >= _MAX_KEY or n >= (1 << 31):  # graph.py:69-71
            raise E.ConfigError(f"unsupported vertex count {num_vertices}")
        lo, hi = (float(x) for x in density_bounds)
        if not 0.0 < lo < hi <= 1.0:
            raise E.ConfigError(f"density bounds must satisfy 0 < lo < hi <= 1, got {density_bounds}")
        seg = int(segment_slots)
        if seg < 2 or int(hi * seg) < 1 or int(hi * seg) >= seg:
            raise E.ConfigError(f"segment_slots={segment_slots} does not fit density bounds {density_bounds}")
        self.segment_slots, self.density_bounds = seg, (lo, hi)
        if slack is None:
            slack = max(0.25, 1.0 / hi - 1.0)
        self.lib = _lib.load()
        self.dev = _device(device)
        self.n = n
        self.slack = float(slack)
        self.min_slack = int(min_slack)
        self.reserve = reserve
        self.ws = torch.empty(0, dtype=torch.uint8, device=self.dev)
        self.batch = DeviceBatch(1024, self.dev, n)
        self.m_hint = 0
        self.compactions = 0  # rebuilds since construction (arena full / explicit)
        # vertex sharding (shard.py): this graph holds the edges whose dst it owns
        self.part_rank, self.part_count = 0, 1
        self._build(np.zeros(0, np.int32), np.zeros(0, np.int32), None)

    # ---------------------------------------------------------------- build
    def _reserve_for(self, m: int) -> int:
        return int(self.reserve) if self.reserve is not None else max(1 << 16, m // 2 + 8 * self.batch.cap)

    def _slots_for(self, lens: torch.Tensor) -> int:
        out = torch.zeros(2, dtype=torch.int64, device=self.dev)
        ws = torch.empty(self.lib.rtec_build_workspace_bytes(self.n, 1), dtype=torch.uint8, device=self.dev)
        _lib.check(self.lib.rtec_graph_slots_needed(_lib.ptr(lens), self.n, self.slack, self.min_slack,
                                                    _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_handle()),
                   "slots_needed")
        return int(out[0].item())

    def _build(self, src, dst, ts):
        dev, n = self.dev, self.n
        m = int(len(src))
        s_t = torch.as_tensor(np.asarray(src, np.int32), device=dev)
        d_t = torch.as_tensor(np.asarray(dst, np.int32), device=dev)
        ts_t = None if ts is None else torch.as_tensor(np.asarray(ts, np.int64), device=dev)
        self._build_tensors(s_t, d_t, ts_t)

    def _build_tensors(self, s_t, d_t, ts_t):
        dev, n, lib = self.dev, self.n, self.lib
        m = int(s_t.numel())
        st = _lib.stream_handle()
        err = torch.full((1,), -1, dtype=torch.int64, device=dev)
        out_deg = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        in_deg = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.rtec_graph_count(_lib.ptr(s_t), _lib.ptr(d_t), m, n, _lib.ptr(out_deg), _lib.ptr(in_deg),
                                        _lib.ptr(err), st), "from_edges")
        _lib.raise_err(err.item(), "from_edges", {1: "edge endpoint outside vertex range"})
        reserve = self._reserve_for(m)
        self.out = _Adj(n, self._slots_for(out_deg) + reserve, dev, True)
        self.inn = _Adj(n, self._slots_for(in_deg) + reserve, dev, False)
        self.out_deg, self.in_deg = out_deg, in_deg
        self.out_deg_prev, self.in_deg_prev = out_deg.clone(), in_deg.clone()
        self.num_edges_t = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(lib.rtec_build_workspace_bytes(n, m), dtype=torch.uint8, device=dev)
        g = self.c()
        _lib.check(lib.rtec_graph_build(C.byref(g), _lib.ptr(s_t), _lib.ptr(d_t), _lib.ptr(ts_t), m, self.slack,
                                        self.min_slack, _lib.ptr(err), _lib.ptr(ws), ws.numel(), st), "from_edges")
        _lib.raise_err(err.item(), "from_edges", {2: "duplicate edges in bulk load"})
        self.m_hint = m
        self._ensure_ws(self.batch.cap)

    def _ensure_ws(self, B: int, grow: float = 1.0):
        need = int(self.lib.rtec_workspace_bytes(self.n, max(B, 1), max(self.out.slots, self.inn.slots), 1) * grow)
        if self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)

    def c(self) -> _lib.Graph:
        p = _lib.ptr
        return _lib.Graph(self.n, self.out.c(), self.inn.c(), p(self.out_deg), p(self.in_deg), p(self.out_deg_prev),
                          p(self.in_deg_prev), p(self.num_edges_t), self.slack, self.min_slack, self.part_rank,
                          self.part_count)

    @classmethod
    def from_edges(cls, num_vertices: int, edges, **kw) -> "DynamicGraph":
        """Bulk load from (src, dst) / (src, dst, ts) tuples or a (src, dst[, ts])
        tuple of arrays; ts defaults to the input index (graph.py:81-121)."""
        g = cls(num_vertices, **kw)
        if isinstance(edges, tuple) and len(edges) in (2, 3) and hasattr(edges[0], "__len__") and not np.isscalar(edges[0]):
            src, dst = np.asarray(edges[0], np.int64), np.asarray(edges[1], np.int64)
            ts = np.asarray(edges[2], np.int64) if len(edges) == 3 else None
        else:
            rows = list(edges)
            if not rows:
                return g
            arr = np.asarray(rows, dtype=np.int64)
            if arr.ndim != 2 or arr.shape[1] not in (2, 3):
                raise E.ConfigError("edges must be (src, dst) or (src, dst, ts) tuples")
            src, dst = arr[:, 0], arr[:, 1]
            ts = arr[:, 2] if arr.shape[1] == 3 else None
        if src.size and (src.min() < 0 or dst.min() < 0 or src.max() >= g.n or dst.max() >= g.n):
            raise E.InvalidVertex("edge endpoint outside vertex range")
        g._build(src, dst, ts)
        return g

    @classmethod
    def from_tensors(cls, num_vertices: int, src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor | None = None,
                     **kw) -> "DynamicGraph":
        """Bulk load from device int32 tensors (no host round trip)."""
        g = cls(num_vertices, **kw)
        g._build_tensors(src.to(g.dev, torch.int32).contiguous(), dst.to(g.dev, torch.int32).contiguous(),
                         None if ts is None else ts.to(g.dev, torch.int64).contiguous())
        return g

    # ---------------------------------------------------------------- queries
    @property
    def num_vertices(self) -> int:
        return self.n

    @property
    def num_edges(self) -> int:
        return int(self.num_edges_t.item())

    @property
    def in_degrees(self) -> np.ndarray:
        return self.in_deg[: self.n].cpu().numpy().astype(np.int64)

    @property
    def out_degrees(self) -> np.ndarray:
        return self.out_deg[: self.n].cpu().numpy().astype(np.int64)

    def _check(self, v: int) -> None:  # graph.py:233-235
        if not (0 <= v < self.n):
            raise E.InvalidVertex(f"vertex {v} outside [0, {self.n})")

    def in_degree(self, v: int) -> int:
        self._check(v)
        return int(self.in_deg[v].item())

    def out_degree(self, v: int) -> int:
        self._check(v)
        return int(self.out_deg[v].item())

    def _run(self, adj: _Adj, v: int) -> np.ndarray:
        b = int(adj.beg[v].item())
        L = int(adj.len[v].item())
        return adj.nbr[b:b + L].cpu().numpy().astype(np.int64)

    def in_neighbors(self, v: int) -> np.ndarray:  # graph.py:155-159
        self._check(v)
        return self._run(self.inn, v)

    def out_neighbors(self, v: int) -> np.ndarray:  # graph.py:161-164
        self._check(v)
        return self._run(self.out, v)

    def has_edge(self, src: int, dst: int) -> bool:  # graph.py:150-153
        self._check(src)
        self._check(dst)
        run = self._run(self.out, src)
        i = np.searchsorted(run, dst)
        return bool(i < run.size and run[i] == dst)

    def _export(self, adj: _Adj, with_ts: bool):
        m = self.num_edges
        v = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
        w = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
        t = torch.empty(max(m, 1), dtype=torch.int64, device=self.dev) if with_ts else None
        a = adj.c()
        _lib.check(self.lib.rtec_adj_export(self.n, C.byref(a), _lib.ptr(v), _lib.ptr(w), _lib.ptr(t),
                                            _lib.ptr(self.ws), self.ws.numel(), _lib.stream_handle()), "edges")
        v, w = v[:m].cpu().numpy().astype(np.int64), w[:m].cpu().numpy().astype(np.int64)
        return v, w, (t[:m].cpu().numpy() if with_ts else None)

    def edges(self):
        """All edges as (src, dst, ts) arrays sorted by (src, dst) (graph.py:166-170)."""
        return self._export(self.out, True)

    def in_edges(self):
        """(dst, src) pairs sorted by (dst, src): the in-adjacency, for consistency checks."""
        v, w, _ = self._export(self.inn, False)
        return v, w

    def copy(self) -> "DynamicGraph":  # graph.py:172-180
        s, d, t = self.edges()
        g = DynamicGraph(self.n, segment_slots=self.segment_slots, density_bounds=self.density_bounds, device=self.dev,
                         slack=self.slack, min_slack=self.min_slack, reserve=self.reserve)
        g._build(s, d, t)
        return g

    # ---------------------------------------------------------------- compaction
    def compact(self, min_reserve: int = 0):
        """Rebuild both adjacencies with fresh slack (replaces PMA rebalance, pma.py:304-326)."""
        st = _lib.stream_handle()
        m = self.num_edges
        for name, with_ts in (("out", True), ("inn", False)):
            old = getattr(self, name)
            new = _Adj(self.n, self._slots_for(old.len) + max(self._reserve_for(m), int(min_reserve)), self.dev, with_ts)
            ws = torch.empty(self.lib.rtec_build_workspace_bytes(self.n, 1), dtype=torch.uint8, device=self.dev)
            a_old, a_new = old.c(), new.c()
            _lib.check(self.lib.rtec_adj_compact(self.n, C.byref(a_old), C.byref(a_new), self.slack, self.min_slack,
                                                 _lib.ptr(ws), ws.numel(), st), "compact")
            setattr(self, name, new)
        self.compactions += 1
        self._ensure_ws(self.batch.cap)

    # ---------------------------------------------------------------- mutation
    def stage(self, op, src, dst, ts) -> int:
        """Copy one batch into the device staging buffers; returns B."""
        B = int(len(src))
        if B > self.batch.cap:
            self.batch = DeviceBatch(max(B, 2 * self.batch.cap), self.dev, self.n)
            self._ensure_ws(self.batch.cap)
        b = self.batch
        if B:
            for dst_t, arr, dt in ((b.op, op, np.uint8), (b.src, src, np.int32), (b.dst, dst, np.int32),
                                   (b.ts, ts, np.int64)):
                if isinstance(arr, torch.Tensor):
                    if arr.dtype != dst_t.dtype:
                        raise E.ShapeError(f"batch tensor dtype {arr.dtype} != {dst_t.dtype}")
                    dst_t[:B].copy_(arr, non_blocking=True)
                else:
                    if dt == np.int32:
                        arr = _i32_ids(arr)
                    dst_t[:B].copy_(torch.from_numpy(np.ascontiguousarray(arr, dt)))
        return B

    def apply_staged(self, B: int, phase: int = 3) -> None:
        """Enqueue rtec_batch_apply on the staged batch (no host sync).  phase 1
        validates + plans (no mutation), 2 mutates, 3 both."""
        if phase & 1:
            self._gc, self._bc = self.c(), self.batch.c()  # kept alive for later calls of the same batch
        g, b = self._gc, self._bc
        p = _lib.ptr
        bb = self.batch
        _lib.check(self.lib.rtec_batch_apply_phase(C.byref(g), C.byref(b), p(bb.src), p(bb.dst), p(bb.op), p(bb.ts),
                                                   B, phase, p(self.ws), self.ws.numel(), _lib.stream_handle()),
                   "apply_batch")

    def commit(self) -> None:
        g, b = self.c(), self.batch.c()
        _lib.check(self.lib.rtec_batch_commit(C.byref(g), C.byref(b), _lib.stream_handle()), "commit")

    def batch_error(self) -> int:
        return int(self.batch.err.item()) & _lib.ERR_OK

    def read_result(self, B: int):
        """(status u8[B], deltas int64[k,5]) of the last applied batch (syncs)."""
        b = self.batch
        status = b.status[:B].cpu().numpy().copy()
        k = int(b.n_delta.item())
        deltas = np.stack([t[:k].cpu().numpy().astype(np.int64) for t in b.d], axis=1) if k else np.zeros((0, 5), np.int64)
        return status, deltas

    _ERR_MSG = {1: "vertex outside the vertex range", 2: "batch not coalesced: duplicate edge"}

    def apply_arrays(self, op, src, dst, ts, *, commit: bool = True):
        """Array form of apply_batch: returns (status, deltas) host arrays."""
        B = self.stage(op, src, dst, ts)
        for attempt in range(4):
            self.apply_staged(B)
            word = self.batch_error()
            d = _lib.decode_err(word)
            if d is not None and d[0] == _lib.ARENA_FULL:
                self.compact(min_reserve=(16 * B + 4096) * 4 ** attempt)
                self._ensure_ws(self.batch.cap, grow=2.0 ** (attempt + 1))
                continue
            _lib.raise_err(word, "apply_batch", self._ERR_MSG)
            break
        else:
            raise E.NativeError("apply_batch: arena still full after compaction")
        res = self.read_result(B)
        if commit:
            self.commit()
        return res

    def apply_batch(self, batch: Sequence[EdgeUpdate]) -> ApplyResult:
        """Apply a coalesced batch atomically (graph.py:184-231)."""
        batch = list(batch)
        op, src, dst, ts = updates_to_arrays(batch)
        status, deltas = self.apply_arrays(op, src, dst, ts)
        applied = tuple(u for u, s in zip(batch, status) if s)
        rejected = tuple(u for u, s in zip(batch, status) if not s)
        dd = tuple(DegreeDelta(*map(int, r)) for r in deltas)
        return ApplyResult(applied, rejected, dd)


# ---- batch helpers (graph.py:241-266) ----


def coalesce_arrays(op, src, dst, ts, device=None):
    """coalesce_batch on arrays, on the device (graph.py:241-260)."""
    lib = _lib.load()
    dev = _device(device)
    B = int(len(src))
    if B == 0:
        z = np.zeros(0, np.int64)
        return z.astype(np.uint8), z, z, z
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dt), device=dev)  # noqa: E731
    s_t, d_t, o_t, ts_t = t(src, np.int32), t(dst, np.int32), t(op, np.uint8), t(ts, np.int64)
    os_, od_, oo_, ot_ = (torch.empty(B, dtype=x, device=dev) for x in (torch.int32, torch.int32, torch.uint8, torch.int64))
    n_out = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(lib.rtec_build_workspace_bytes(1, B) + 64 * B, dtype=torch.uint8, device=dev)
    p = _lib.ptr
    _lib.check(lib.rtec_batch_coalesce(p(s_t), p(d_t), p(o_t), p(ts_t), B, p(os_), p(od_), p(oo_), p(ot_), p(n_out),
                                       p(ws), ws.numel(), _lib.stream_handle()), "coalesce_batch")
    k = int(n_out.item())
    return (oo_[:k].cpu().numpy(), os_[:k].cpu().numpy().astype(np.int64), od_[:k].cpu().numpy().astype(np.int64),
            ot_[:k].cpu().numpy())


def coalesce_batch(batch: Sequence[EdgeUpdate]) -> list:
    """Net effect per edge; survivors keep the first establishing ts, in order
    of first appearance (graph.py:241-260)."""
    batch = list(batch)
    if not batch:
        return []
    op, src, dst, ts = updates_to_arrays(batch)
    for a in (src, dst):
        if a.size and (a.min() < -(1 << 31) or a.max() >= (1 << 31)):
            raise E.InvalidVertex("vertex id beyond int32")
    o, s, d, t = coalesce_arrays(op, src, dst, ts)
    ops = (UpdateOp.INSERT, UpdateOp.DELETE)
    return [EdgeUpdate(ops[int(a)], int(b), int(c), int(e)) for a, b, c, e in zip(o, s, d, t)]


def invert_batch(batch: Sequence[EdgeUpdate]) -> list:
    """graph.py:263-266: swap inserts and deletes."""
    flip = {UpdateOp.INSERT: UpdateOp.DELETE, UpdateOp.DELETE: UpdateOp.INSERT}
    return [EdgeUpdate(flip[u.op], u.src, u.dst, u.ts) for u in batch]


def _parse_update(path: str, lineno: int, text: str) -> EdgeUpdate:
    """One 'op,src,dst,ts' record of an edge-stream file (graph.py:269-293 format)."""
    fields = text.split(",")
    op = {"+": UpdateOp.INSERT, "-": UpdateOp.DELETE}.get(fields[0]) if len(fields) == 4 else None
    if op is None:
        raise E.ConfigError(f"{path}:{lineno}: malformed update line {text!r}")
    try:
        ids = [int(f) for f in fields[1:]]
    except ValueError as exc:
        raise E.ConfigError(f"{path}:{lineno}: non-integer field in {text!r}") from exc
    return EdgeUpdate(op, *ids)


def read_stream(path: str) -> list:
    """Edge-stream text file: one 'op,src,dst,ts' update per line; blank lines and
    '#' comments skipped; a malformed record raises ConfigError naming path:line."""
    with open(path, "r", encoding="ascii") as fh:
        lines = [(k, ln.strip()) for k, ln in enumerate(fh, start=1)]
    return [_parse_update(path, k, t) for k, t in lines if t and not t.startswith("#")]


def write_stream(path: str, updates: Iterable[EdgeUpdate]) -> None:
    """Inverse of read_stream (one record per line, ASCII)."""
    recs = "".join("%s,%d,%d,%d\n" % (u.op.value, u.src, u.dst, u.ts) for u in updates)
    with open(path, "w", encoding="ascii") as fh:
        fh.write(recs)
