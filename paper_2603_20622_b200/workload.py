"""Seeded synthetic workloads: graphs, update streams, features.

The reference's harness (generators + stream splitter) was
never shipped; this restates the parts the benchmark needs:

- `chung_lu_edges`: power-law Chung-Lu graph, weights w_i ∝ (i+1)^-alpha,
  independent random permutations for the source and destination roles,
  unique directed edges (self-loops allowed), exactly m edges.
- `rmat_edges`: R-MAT (a, b, c, d) on 2^scale ids, relabelled and trimmed.
- `UpdateStream`: base = first (1 - holdout) of the edges; every batch is B/2
  inserts drawn without replacement from the hold-out plus B/2 deletes drawn
  uniformly from the live edges, shuffled,
  already coalesced (no repeated (src, dst) inside a batch).

Host-side setup code (numpy); not on the timed path.
"""

from __future__ import annotations

import numpy as np

OP_INSERT = 0
OP_DELETE = 1


def _unique_fill(sample, n, m, rng, max_rounds=64):
    """Draw key batches until m unique (src*n+dst) keys exist; keep first-seen order."""
    keys = np.empty(0, np.uint64)
    need = m
    for _ in range(max_rounds):
        s, d = sample(int(need * 1.15) + 1024)
        k = s.astype(np.uint64) * np.uint64(n) + d.astype(np.uint64)
        keys = np.concatenate([keys, k])
        _, first = np.unique(keys, return_index=True)
        first.sort()
        keys = keys[first]
        if keys.size >= m:
            keys = keys[:m]
            break
        need = m - keys.size
    else:
        raise RuntimeError(f"could not draw {m} unique edges on {n} vertices")
    return (keys // np.uint64(n)).astype(np.int64), (keys % np.uint64(n)).astype(np.int64)


def chung_lu_edges(n: int, m: int, alpha: float = 0.8, seed: int = 0):
    rng = np.random.default_rng(seed)
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-alpha)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm_s = rng.permutation(n)
    perm_d = rng.permutation(n)

    def sample(k):
        a = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), n - 1)
        b = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), n - 1)
        return perm_s[a], perm_d[b]

    return _unique_fill(sample, n, m, rng)


def rmat_edges(n: int, m: int, a=0.57, b=0.19, c=0.19, seed: int = 0):
    rng = np.random.default_rng(seed)
    scale = max(1, int(np.ceil(np.log2(max(n, 2)))))
    cp = np.cumsum(np.array([a, b, c, 1.0 - a - b - c]))
    perm = rng.permutation(1 << scale)  # relabel, then fold ids >= n back by modulus

    def sample(k):
        s = np.zeros(k, np.int64)
        d = np.zeros(k, np.int64)
        for bit in range(scale):
            q = np.minimum(np.searchsorted(cp, rng.random(k), side="right"), 3)
            s |= ((q >> 1) & 1) << bit
            d |= (q & 1) << bit
        return perm[s] % n, perm[d] % n

    return _unique_fill(sample, n, m, rng)


def features(n: int, d: int, seed: int = 1) -> np.ndarray:
    """X ~ U(-1, 1), float32; the oracle reads the same values."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (n, d)).astype(np.float32)


class UpdateStream:
    """Base graph + mixed insert/delete batches over a fixed edge universe."""

    def __init__(self, src, dst, holdout: float = 0.1, seed: int = 0):
        src = np.asarray(src, np.int64)
        dst = np.asarray(dst, np.int64)
        m = src.size
        self.m_total = m
        self.src_all, self.dst_all = src, dst
        nb = int(round(m * (1.0 - holdout)))
        self.base_ids = np.arange(nb)
        self.hold_ids = np.arange(nb, m)
        self.live = np.zeros(m, bool)
        self.live[:nb] = True
        self._hold_ptr = 0
        self._seed = seed
        self._batch = 0
        self._hold_perm = np.random.default_rng(seed + 1_000_003).permutation(self.hold_ids)

    def base(self):
        ids = self.base_ids
        return self.src_all[ids], self.dst_all[ids], ids.astype(np.int64)

    def next_batch(self, B: int):
        """(op uint8, src int64, dst int64, ts int64); seed 2 + batch index."""
        rng = np.random.default_rng(2 + self._batch)
        self._batch += 1
        n_ins = min(B // 2, self._hold_perm.size - self._hold_ptr)
        ins = self._hold_perm[self._hold_ptr:self._hold_ptr + n_ins]
        self._hold_ptr += n_ins
        live_ids = np.flatnonzero(self.live)
        n_del = min(B - n_ins, live_ids.size)
        dels = live_ids[rng.choice(live_ids.size, n_del, replace=False)]
        self.live[dels] = False
        self.live[ins] = True
        ids = np.concatenate([ins, dels])
        op = np.concatenate([np.full(n_ins, OP_INSERT, np.uint8), np.full(n_del, OP_DELETE, np.uint8)])
        perm = rng.permutation(ids.size)
        ids, op = ids[perm], op[perm]
        ts = np.where(op == OP_INSERT, ids, self.m_total + self._batch).astype(np.int64)
        return op, self.src_all[ids], self.dst_all[ids], ts
