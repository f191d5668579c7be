"""Seeded synthetic workloads: graphs, update streams, features.

The reference's harness (generators + stream splitter) was
never shipped; this restates the parts the benchmark needs:

- `chung_lu_edges`: power-law Chung-Lu graph, weights w_i ∝ (i+1)^-alpha,
  independent random permutations for the source and destination roles,
  unique directed edges (self-loops allowed), exactly m edges.
- `rmat_edges`: R-MAT (a, b, c, d) on 2^scale ids, relabelled, folded to n.
- `UpdateStream`: base = first (1 - holdout) of the edges; every batch is B/2
  inserts drawn without replacement from the hold-out plus B/2 deletes drawn
  uniformly from the live edges, shuffled,
  already coalesced (no repeated (src, dst) inside a batch).

Randomness comes from a counter-based splitmix64 hash, so numpy, torch-CPU
and torch-CUDA produce bit-identical graphs (the CPU oracle and the GPU
engine see the same input; generation on the GPU takes ~1 s at 62M edges).
Host-side setup code; not on the timed path.
"""

from __future__ import annotations

import numpy as np

OP_INSERT = 0
OP_DELETE = 1

_M64 = (1 << 64) - 1
_C1, _C2, _C3 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _s64(c):  # unsigned 64-bit constant as a signed int64 (torch has no uint64 arithmetic)
    return c - (1 << 64) if c >= (1 << 63) else c


def _hash_u53(seed: int, stream: int, start: int, count: int, device=None):
    """splitmix64(seed, stream, index) -> uniform [0, 1) doubles (torch float64)."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cpu")
    x = torch.arange(start, start + count, dtype=torch.int64, device=dev)
    base = (seed * 0x100000001B3 + stream * 0x51ED27) & _M64
    x = x + _s64((base + _C1) & _M64)

    def lsr(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)

    z = x
    z = (z ^ lsr(z, 30)) * _s64(_C2)
    z = (z ^ lsr(z, 27)) * _s64(_C3)
    z = z ^ lsr(z, 31)
    return lsr(z, 11).to(torch.float64) * (1.0 / (1 << 53))


def _perm(seed: int, stream: int, n: int, device=None):
    import torch

    return torch.argsort(_hash_u53(seed, stream, 0, n, device), stable=True)


def _unique_fill(sample, n: int, m: int, device, max_rounds: int = 64):
    """Draw until m unique keys src*n+dst exist; keep first-drawn order."""
    import torch

    keys = torch.empty(0, dtype=torch.int64, device=device)
    drawn = 0
    need = m
    for _ in range(max_rounds):
        k = int(need * 1.15) + 1024
        s, d = sample(drawn, k)
        drawn += k
        keys = torch.cat([keys, s * n + d])
        uniq, inv = torch.unique(keys, return_inverse=True)
        first = torch.full((uniq.numel(),), keys.numel(), dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(keys.numel(), device=device), reduce="amin")
        keys = keys[torch.sort(first).values]
        if keys.numel() >= m:
            keys = keys[:m]
            break
        need = m - keys.numel()
    else:
        raise RuntimeError(f"could not draw {m} unique edges on {n} vertices")
    return keys // n, keys % n


def chung_lu_edges(n: int, m: int, alpha: float = 0.8, seed: int = 0, device=None, as_numpy: bool = True):
    import torch

    dev = torch.device(device) if device is not None else torch.device("cpu")
    w = (torch.arange(n, dtype=torch.float64, device=dev) + 1.0) ** (-alpha)
    cdf = torch.cumsum(w, 0)
    cdf = cdf / cdf[-1]
    perm_s = _perm(seed, 11, n, dev)
    perm_d = _perm(seed, 12, n, dev)

    def sample(off, k):
        a = torch.searchsorted(cdf, _hash_u53(seed, 21, off, k, dev), right=True).clamp_(max=n - 1)
        b = torch.searchsorted(cdf, _hash_u53(seed, 22, off, k, dev), right=True).clamp_(max=n - 1)
        return perm_s[a], perm_d[b]

    s, d = _unique_fill(sample, n, m, dev)
    return (s.cpu().numpy(), d.cpu().numpy()) if as_numpy else (s, d)


def rmat_edges(n: int, m: int, a=0.57, b=0.19, c=0.19, seed: int = 0, device=None, as_numpy: bool = True):
    import torch

    dev = torch.device(device) if device is not None else torch.device("cpu")
    scale = max(1, int(np.ceil(np.log2(max(n, 2)))))
    cp = torch.tensor([a, a + b, a + b + c], dtype=torch.float64, device=dev)
    perm = _perm(seed, 31, 1 << scale, dev)

    def sample(off, k):
        s = torch.zeros(k, dtype=torch.int64, device=dev)
        d = torch.zeros(k, dtype=torch.int64, device=dev)
        for bit in range(scale):
            q = torch.searchsorted(cp, _hash_u53(seed, 100 + bit, off, k, dev), right=True)
            s |= ((q >> 1) & 1) << bit
            d |= (q & 1) << bit
        return perm[s] % n, perm[d] % n

    s, d = _unique_fill(sample, n, m, dev)
    return (s.cpu().numpy(), d.cpu().numpy()) if as_numpy else (s, d)


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
        self.live = np.zeros(m, bool)
        self.live[:nb] = True
        self._hold_ptr = 0
        self._batch = 0
        self._hold_perm = np.random.default_rng(seed + 1_000_003).permutation(np.arange(nb, m))

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
