"""ctypes wrapper of oracle/librtec_cpu.so (C + OpenMP oracle port) -- TEST / BASELINE INFRASTRUCTURE ONLY.

Same algorithms as oracle/engine.py (pinned to the reference), for gcn /
graphsage / gin in f64 with every host thread; used by tests (parity with the
numpy oracle) and by bench.py's CPU leg.  Built by `build()` below (also
called from __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rtec_cpu.c")
LIB = os.path.join(HERE, "librtec_cpu.so")
MODELS = {"gcn": 0, "graphsage": 1, "gin": 2}


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB, "-lm"],
                       check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        L.rc_create.restype = P
        L.rc_create.argtypes = [C.c_int64, C.c_int64, P, P, P, C.c_int, C.c_int, P, P, P, C.c_double, P]
        L.rc_step.restype = C.c_int
        L.rc_step.argtypes = [P, C.c_int64, P, P, P, P, P, P, P]
        L.rc_get_h.argtypes = [P, C.c_int, P]
        L.rc_free.argtypes = [P]
        L.rc_num_edges.restype = C.c_int64
        L.rc_num_edges.argtypes = [P]
        L.rc_frontier.argtypes = [P, C.c_int, P, P]
        L.rc_threads.restype = C.c_int
        L.rc_get_rows.argtypes = [P, C.c_int, C.c_int, P, C.c_int64, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class CPortEngine:
    """Incremental engine (oracle port) with the reference's f64 weights."""

    def __init__(self, model, n, src, dst, ts, layers_W, layers_W2, dims, X, degree_offset=1.0):
        L = lib()
        self.n, self.dims = int(n), [int(d) for d in dims]
        self._keep = []
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        ts = np.ascontiguousarray(ts if ts is not None else np.arange(src.size), np.int64)
        Ws = [np.ascontiguousarray(w, np.float64) for w in layers_W]
        W2s = [np.ascontiguousarray(w, np.float64) for w in (layers_W2 or [])]
        self._keep += Ws + W2s
        Wp = (C.c_void_p * len(Ws))(*[w.ctypes.data for w in Ws])
        W2p = (C.c_void_p * max(len(W2s), 1))(*([w.ctypes.data for w in W2s] or [None]))
        d = np.asarray(self.dims, np.int32)
        X = np.ascontiguousarray(X, np.float64)
        self.h = L.rc_create(self.n, src.size, _p(src), _p(dst), _p(ts), MODELS[model], len(self.dims) - 1, _p(d),
                             C.cast(Wp, C.c_void_p), C.cast(W2p, C.c_void_p), float(degree_offset), _p(X))
        self.threads = L.rc_threads()

    def step(self, op, src, dst, ts):
        B = len(src)
        op = np.ascontiguousarray(op, np.uint8)
        s = np.ascontiguousarray(np.clip(np.asarray(src, np.int64), -1, 2**31 - 1), np.int32)
        d = np.ascontiguousarray(np.clip(np.asarray(dst, np.int64), -1, 2**31 - 1), np.int32)
        t = np.ascontiguousarray(ts, np.int64)
        status = np.zeros(max(B, 1), np.uint8)
        deltas = np.zeros((max(2 * B, 1), 5), np.int64)
        nd = np.zeros(1, np.int64)
        rc = lib().rc_step(self.h, B, _p(op), _p(s), _p(d), _p(t), _p(status), _p(deltas), _p(nd))
        if rc:
            raise ValueError({1: "InvalidVertex", 2: "ConfigError"}[rc])
        return status[:B], deltas[: int(nd[0])]

    def H(self, l):
        out = np.empty((self.n, self.dims[l]), np.float64)
        lib().rc_get_h(self.h, l, _p(out))
        return out

    def rows(self, kind: str, l: int, ids) -> np.ndarray:
        """Rows `ids` of H^l (kind 'H') or of the un-normalised aggregate S^l (kind 'S')."""
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.empty((ids.size, self.dims[l]), np.float64)
        lib().rc_get_rows(self.h, 0 if kind == "H" else 1, l, _p(ids), ids.size, _p(out))
        return out

    def frontier(self, l):
        a, b = np.zeros(1, np.int64), np.zeros(1, np.int64)
        lib().rc_frontier(self.h, l, _p(a), _p(b))
        return int(a[0]), int(b[0])

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rc_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
