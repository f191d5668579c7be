"""Oracle restatement of the reference dynamic graph -- TEST INFRASTRUCTURE ONLY.

Restates `streamgnn/graph.py` (reference) semantics over flat sorted arrays:
the out-adjacency is the sorted array of composite keys src*n+dst with a
parallel timestamp array, the in-adjacency the sorted array of dst*n+src
(graph.py:3-14, :73-76).  The PMA layout itself (pma.py) only provides "sorted,
unique, ascending neighbour runs", which a sorted array gives directly.

Update encoding used throughout the oracle and the engine: op 0 = INSERT
("+"), op 1 = DELETE ("-") (graph.py:28-30).
"""

from __future__ import annotations

import numpy as np

OP_INSERT = 0
OP_DELETE = 1

# exception *names* raised by the reference at its boundary (errors.py:10-35)
ERR_INVALID_VERTEX = "InvalidVertex"
ERR_CONFIG = "ConfigError"


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class OracleGraph:
    """DynamicGraph semantics (graph.py:59-235) on sorted uint64 key arrays."""

    def __init__(self, n: int):
        n = int(n)
        if n < 0 or n * n >= (1 << 62):  # graph.py:70-71 (pma.MAX_KEY)
            raise OracleError(ERR_CONFIG, f"unsupported vertex count {n}")
        self.n = n
        self.out_keys = np.empty(0, np.uint64)
        self.out_ts = np.empty(0, np.int64)
        self.in_keys = np.empty(0, np.uint64)
        self.out_deg = np.zeros(n, np.int64)
        self.in_deg = np.zeros(n, np.int64)

    # ---- bulk load: graph.py:81-121 ----
    @classmethod
    def from_edges(cls, n, src, dst, ts=None) -> "OracleGraph":
        g = cls(n)
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        if src.size == 0:
            return g
        ts = np.arange(src.size, dtype=np.int64) if ts is None else np.asarray(ts, np.int64)  # :100
        if src.min() < 0 or dst.min() < 0 or src.max() >= n or dst.max() >= n:  # :101-102
            raise OracleError(ERR_INVALID_VERTEX, "edge endpoint outside vertex range")
        nn = np.uint64(n)
        ok = src.astype(np.uint64) * nn + dst.astype(np.uint64)
        order = np.argsort(ok, kind="stable")  # :104
        oks = ok[order]
        if oks.size > 1 and np.any(oks[1:] == oks[:-1]):  # :106-107
            raise OracleError(ERR_CONFIG, "duplicate edges in bulk load")
        g.out_keys = oks
        g.out_ts = ts[order]
        g.in_keys = np.sort(dst.astype(np.uint64) * nn + src.astype(np.uint64))  # :108
        np.add.at(g.out_deg, src, 1)  # :118-119
        np.add.at(g.in_deg, dst, 1)
        return g

    def copy(self) -> "OracleGraph":  # graph.py:172-180
        g = OracleGraph.__new__(OracleGraph)
        g.n = self.n
        g.out_keys = self.out_keys.copy()
        g.out_ts = self.out_ts.copy()
        g.in_keys = self.in_keys.copy()
        g.out_deg = self.out_deg.copy()
        g.in_deg = self.in_deg.copy()
        return g

    # ---- queries: graph.py:124-170 ----
    @property
    def num_edges(self) -> int:
        return int(self.out_keys.size)

    def _run(self, keys, v):
        nn = np.uint64(self.n)
        lo = np.searchsorted(keys, np.uint64(v) * nn)
        hi = np.searchsorted(keys, np.uint64(v + 1) * nn)
        return (keys[lo:hi] % nn).astype(np.int64)

    def in_neighbors(self, v: int) -> np.ndarray:  # graph.py:155-159
        return self._run(self.in_keys, v)

    def out_neighbors(self, v: int) -> np.ndarray:  # graph.py:161-164
        return self._run(self.out_keys, v)

    def has_edge(self, s: int, d: int) -> bool:  # graph.py:150-153
        k = np.uint64(s) * np.uint64(self.n) + np.uint64(d)
        i = np.searchsorted(self.out_keys, k)
        return bool(i < self.out_keys.size and self.out_keys[i] == k)

    def edges(self):  # graph.py:166-170: sorted by (src, dst) with ts
        nn = np.uint64(max(self.n, 1))
        return (
            (self.out_keys // nn).astype(np.int64),
            (self.out_keys % nn).astype(np.int64),
            self.out_ts.copy(),
        )

    def in_csr(self):
        """(indptr, sources) of the in-adjacency; runs ascending by source."""
        nn = np.uint64(max(self.n, 1))
        dst = (self.in_keys // nn).astype(np.int64)
        indptr = np.zeros(self.n + 1, np.int64)
        np.cumsum(np.bincount(dst, minlength=self.n), out=indptr[1:])
        return indptr, (self.in_keys % nn).astype(np.int64)

    def out_csr(self):
        nn = np.uint64(max(self.n, 1))
        src = (self.out_keys // nn).astype(np.int64)
        indptr = np.zeros(self.n + 1, np.int64)
        np.cumsum(np.bincount(src, minlength=self.n), out=indptr[1:])
        return indptr, (self.out_keys % nn).astype(np.int64)

    # ---- mutation: graph.py:184-231 ----
    def apply_batch(self, op, src, dst, ts):
        """Apply a coalesced batch.

        Returns (status, deltas): status[i] = 1 if update i applied, 0 if
        rejected (duplicate insert / absent delete, graph.py:209-219); deltas
        = int64[k, 5] rows (vertex, old_in, new_in, old_out, new_out) for
        every touched vertex whose degrees changed, ascending (graph.py:225-230).
        Validation (range -> InvalidVertex, repeated edge -> ConfigError) runs
        over the whole batch, in batch order, before any mutation (:192-198).
        """
        op = np.asarray(op, np.int64)
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        ts = np.asarray(ts, np.int64)
        n = self.n
        B = src.size
        if B == 0:
            return np.zeros(0, np.uint8), np.zeros((0, 5), np.int64)
        # -- validation pass (graph.py:192-198): first offending position wins
        bad_range = (src < 0) | (src >= n) | (dst < 0) | (dst >= n)
        first_bad = int(np.argmax(bad_range)) if bad_range.any() else B
        nn = np.uint64(max(n, 1))
        keys = np.where(bad_range, 0, src).astype(np.uint64) * nn + np.where(bad_range, 0, dst).astype(np.uint64)
        order = np.argsort(keys, kind="stable")
        ks = keys[order]
        dup_sorted = np.zeros(B, bool)
        dup_sorted[1:] = ks[1:] == ks[:-1]
        dup = np.zeros(B, bool)
        dup[order] = dup_sorted
        dup &= ~bad_range
        # a duplicate only counts if its earlier twin was itself range-valid (always
        # true here: an invalid twin would have raised first)
        first_dup = int(np.argmax(dup)) if dup.any() else B
        if first_bad < B or first_dup < B:
            if first_bad <= first_dup:
                raise OracleError(ERR_INVALID_VERTEX, f"vertex outside [0, {n})")
            raise OracleError(ERR_CONFIG, "batch not coalesced")
        # -- old degrees of every endpoint, captured before mutation (:205-207)
        touched = np.unique(np.concatenate([src, dst]))
        old_in = self.in_deg[touched].copy()
        old_out = self.out_deg[touched].copy()
        # -- existence probe against the pre-batch graph; keys are unique so
        #    the sequential loop of :202-224 reduces to independent probes
        pos = np.searchsorted(self.out_keys, keys)
        exists = np.zeros(B, bool)
        inb = pos < self.out_keys.size
        exists[inb] = self.out_keys[pos[inb]] == keys[inb]
        ins = (op == OP_INSERT) & ~exists
        dele = (op == OP_DELETE) & exists
        status = (ins | dele).astype(np.uint8)
        # -- mutate out (with ts) and in adjacencies
        keep = ~np.isin(self.out_keys, keys[dele])
        ok_all = np.concatenate([self.out_keys[keep], keys[ins]])
        ts_all = np.concatenate([self.out_ts[keep], ts[ins]])
        o = np.argsort(ok_all, kind="stable")
        self.out_keys, self.out_ts = ok_all[o], ts_all[o]
        in_k = dst.astype(np.uint64) * nn + src.astype(np.uint64)
        keep_in = ~np.isin(self.in_keys, in_k[dele])
        self.in_keys = np.sort(np.concatenate([self.in_keys[keep_in], in_k[ins]]))
        np.add.at(self.out_deg, src[ins], 1)
        np.add.at(self.in_deg, dst[ins], 1)
        np.add.at(self.out_deg, src[dele], -1)
        np.add.at(self.in_deg, dst[dele], -1)
        new_in = self.in_deg[touched]
        new_out = self.out_deg[touched]
        ch = (old_in != new_in) | (old_out != new_out)
        deltas = np.stack([touched[ch], old_in[ch], new_in[ch], old_out[ch], new_out[ch]], axis=1)
        return status, deltas.astype(np.int64)


def coalesce_batch(op, src, dst, ts):
    """Net effect per (src, dst): graph.py:241-260.

    Same ops collapse (the first event's ts survives), opposite ops cancel;
    survivors come out in order of the key's FIRST appearance in the batch.
    Returns (op, src, dst, ts) arrays.
    """
    order: list = []
    state: dict = {}
    for i in range(len(src)):
        key = (int(src[i]), int(dst[i]))
        u = (int(op[i]), key[0], key[1], int(ts[i]))
        if key not in state:
            state[key] = u
            order.append(key)
        else:
            cur = state[key]
            if cur is None:
                state[key] = u
            elif cur[0] != u[0]:
                state[key] = None
    out = [state[k] for k in order if state[k] is not None]
    if not out:
        z = np.zeros(0, np.int64)
        return z.astype(np.uint8), z, z, z
    a = np.asarray(out, np.int64)
    return a[:, 0].astype(np.uint8), a[:, 1], a[:, 2], a[:, 3]


def invert_batch(op, src, dst, ts):
    """graph.py:263-266: swap inserts and deletes."""
    op = np.asarray(op, np.uint8)
    return (1 - op).astype(np.uint8), np.asarray(src), np.asarray(dst), np.asarray(ts)
