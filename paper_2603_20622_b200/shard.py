"""Vertex-sharded incremental engine with a ghost-row store: one process per GPU
(SURVEY §8(e)).

The reference is single-process CPU code and the paper offloads
the historical embeddings to host memory.  Here they are
sharded over the GPUs' HBM, destination-owned, with no replicas:

- owner(v) = v mod P.  Rank p holds every edge whose dst it owns (in- and
  out-runs) over LOCAL ids: [0, n_own) its owned vertices (local i <-> global
  p + P i), then ghosts -- the sources with an out-edge into the shard.  Every
  per-vertex array of the rank is sized by its local id capacity (owned +
  ghosts + headroom), and the layer kernels run unchanged on the local graph.
- Ghost rows of the layer inputs H^0..H^{L-1} (and GAT's Z / el / er) are kept
  coherent by their owner: `peers[v]` (bit q = rank q holds a ghost of v) is
  built at load time and extended by each batch's inserts (ghost admission: the
  owner ships the new ghost's pre-batch rows and global out-degree).  After
  layer l every rank sends each changed owned row only to the ranks in its
  `peers` mask (a targeted all-to-all over NCCL); receivers overwrite the ghost
  row and keep the overwritten (pre-batch) one as the exchanged DeltaLog that
  layer l+1 retracts with.
- Global out-degrees (GCN's 1/sqrt(d_out(u)+off), models.py:98-99, and the F1
  Dg seed) are kept for every local vertex and updated from the globally
  applied set (per-update status MAX-all-reduced; each update has one owner).
  Every rank validates the whole batch (identical InvalidVertex / ConfigError
  everywhere, before anything mutates: graph.py:192-198); the shard applies its
  own updates in two phases with the ranks' status words combined in between,
  so a full arena anywhere leaves every shard untouched.

Host synchronisations per batch: one after validation / admission / localisation
(error word and sizes), one between the apply phases, one per exchanged layer (the
all-to-all row counts NCCL needs on the host), one at the end (status words,
results).  Exchange volume per layer: Σ_{v ∈ V_dst(l)} |peers(v)| rows of
d_{l+1} floats (`exchange_log`).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import errors as E
from .engine import Metrics, RTECEngine, RunResult, _Frontier
from .graph import DynamicGraph
from .models import GAT, GCN, GIN, GRAPHSAGE, PROJECTED

SUM_MODELS = (GCN, GRAPHSAGE, GIN)

_U64 = (1 << 64) - 1
MAX_WORLD = 32  # RTEC_SHARD_MAX_WORLD: peers masks are 32-bit


def owner_of(v, world: int):
    """Partition function of the shards (owner(v) = v mod P)."""
    return v % world


def owned_count(n: int, rank: int, world: int) -> int:
    """|{v < n : v mod world == rank}|."""
    return max((n - rank + world - 1) // world, 0)


class Comm:
    """The collectives the sharded engine issues, over torch.distributed (NCCL on
    device tensors; gloo groups -- CPU tests, ranks sharing a GPU -- staged through
    host memory)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = str(dist.get_backend(group))
        self.staged = self.backend != "nccl"

    def all_reduce_(self, t: torch.Tensor, op=dist.ReduceOp.SUM) -> torch.Tensor:
        x = t.cpu() if self.staged and t.is_cuda else t
        dist.all_reduce(x, op=op, group=self.group)
        if x is not t:
            t.copy_(x)
        return t

    def all_gather_ints(self, values, device) -> np.ndarray:
        """[world, k] int64 host array of every rank's k host integers."""
        v = torch.tensor(list(values), dtype=torch.int64, device=torch.device("cpu") if self.staged else device)
        out = [torch.empty_like(v) for _ in range(self.world)]
        dist.all_gather(out, v, group=self.group)
        return torch.stack(out).cpu().numpy()

    def all_gather_var(self, t: torch.Tensor, count: int) -> torch.Tensor:
        """Concatenation over ranks (rank order) of each rank's first `count` rows of t."""
        counts = self.all_gather_ints([count], t.device)[:, 0]
        cap = max(int(counts.max(initial=0)), 1)
        buf = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        if count:
            buf[:count] = t[:count]
        if self.staged:
            buf = buf.cpu()
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return torch.cat([o[: int(c)] for o, c in zip(outs, counts)]).to(t.device)

    def all_to_all_counts(self, send: torch.Tensor) -> torch.Tensor:
        """[world] int64 per-peer counts -> the counts every peer sends here."""
        x = send.cpu() if self.staged else send
        out = torch.empty_like(x)
        dist.all_to_all_single(out, x, group=self.group)
        return out.to(send.device)

    def all_to_all_rows(self, t: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        """Rows of t grouped by destination rank (send_counts[q] rows to q) -> the rows
        received, grouped by source rank."""
        sc, rc = [int(c) for c in send_counts], [int(c) for c in recv_counts]
        shape = (sum(rc),) + tuple(t.shape[1:])
        x = t[: sum(sc)].contiguous()
        if self.staged:
            out = torch.empty(shape, dtype=t.dtype)
            dist.all_to_all_single(out, x.cpu(), rc, sc, group=self.group)
            return out.to(t.device)
        out = torch.empty(shape, dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, x, rc, sc, group=self.group)
        return out


def combine_err_words(words) -> int:
    """Status words of all ranks -> the batch's word: smallest (position, code) wins (unsigned)."""
    return min(int(w) & _U64 for w in words)


def _signed(w: int) -> int:
    return w - (1 << 64) if w >= (1 << 63) else w


def _ptr_array(ptrs):
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    return arr, C.cast(arr, C.c_void_p)


def _int_array(vals, ct=C.c_int32):
    arr = (ct * len(vals))(*[int(v) for v in vals])
    return arr, C.cast(arr, C.c_void_p)


class ShardedRTECEngine(RTECEngine):
    """RTECEngine over this rank's shard of the graph; same step() /
    query() / embeddings() API, collective over the ranks of `comm`."""

    # sum aggregators: the update epilogue writes δ of the owned changed rows and the exchange
    # writes δ of the received ghost rows (no DeltaLog); GAT / GIN-max keep an exchanged DeltaLog
    FUSED_DELTA = True

    def __init__(self, bundle, num_vertices: int, edges, features, comm: Comm, *, max_batch: int | None = None,
                 update: str = "tc", reserve: int | None = None, device=None, exchange_chunk: int = 1 << 20,
                 bootstrap: bool = True, shard_edges: bool = False, ghost_headroom: float = 0.10):
        """edges: (src, dst[, ts]) global edge list (every rank passes the same), or with
        shard_edges=True only this rank's edges (owner(dst) == rank; checkpoint resume).
        features: [n, d0] global, or [n_own, d0] owned rows in owner order."""
        if bundle.model in PROJECTED:  # payload / gate caches are not exchanged between shards
            raise E.UnsupportedModel(f"sharded engine: model {bundle.model!r} not supported")
        if comm.world > MAX_WORLD:
            raise E.ConfigError(f"sharded engine: world size {comm.world} > {MAX_WORLD}")
        self.comm = comm
        P, r = comm.world, comm.rank
        n = int(num_vertices)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

        def as_t(a, dt):
            return (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))).to(dev, dt)

        src, dst = as_t(edges[0], torch.int64), as_t(edges[1], torch.int64)
        ts = (torch.arange(src.numel(), dtype=torch.int64, device=dev) if len(edges) < 3 or edges[2] is None
              else as_t(edges[2], torch.int64))
        if src.numel() and (int(src.min()) < 0 or int(dst.min()) < 0 or int(src.max()) >= n or int(dst.max()) >= n):
            raise E.InvalidVertex("edge endpoint outside vertex range")
        if not shard_edges:
            mine = owner_of(dst, P) == r
            src, dst, ts = src[mine], dst[mine], ts[mine]
        elif src.numel() and bool((owner_of(dst, P) != r).any()):
            raise E.ConfigError("shard_edges: an edge's destination is not owned by this rank")
        self.n_glob, self.n_own = n, owned_count(n, r, P)
        self.exchange_chunk = int(exchange_chunk)
        self.ghost_headroom = float(ghost_headroom)
        self._reserve = reserve
        # local ids: owned (v // P), then ghosts in ascending global id
        gh = torch.unique(src[owner_of(src, P) != r])
        n_loc = self.n_own + gh.numel()
        B0 = int(max_batch or 1024)
        cap = self._cap_for(n_loc, B0)
        self.g2l = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
        self.g2l[r::P] = torch.arange(self.n_own, dtype=torch.int32, device=dev)
        self.g2l[gh] = torch.arange(self.n_own, n_loc, dtype=torch.int32, device=dev)
        self.l2g = torch.full((cap,), -1, dtype=torch.int32, device=dev)
        self.l2g[: self.n_own] = torch.arange(r, n, P, dtype=torch.int32, device=dev)
        self.l2g[self.n_own:n_loc] = gh.to(torch.int32)
        self.n_loc_t = torch.tensor([n_loc], dtype=torch.int64, device=dev)
        self.n_loc = n_loc
        self.admitted = 0
        self.peers = torch.zeros(max(self.n_own, 1), dtype=torch.int32, device=dev)
        g = DynamicGraph.from_tensors(cap, self.g2l[src], self.g2l[dst], ts, device=dev, reserve=reserve)
        # global out-degree of every local vertex: owners sum the shards' local out-degrees
        # (each edge lives in exactly one shard); the same announce builds peers[]
        self.gout = g.out_deg.clone()
        self._announce(g)
        self.gout_prev = self.gout.clone()

        def zi(k, dt=torch.int32):
            return torch.zeros(max(k, 1), dtype=dt, device=dev)

        self.dg_bm = zi((cap + 31) // 32)
        self.bm_touch = zi((self.n_own + 31) // 32)
        self.bm_adm = zi((n + 31) // 32)
        self.sdelta = [zi(2 * B0) for _ in range(5)]
        self.n_sdelta = zi(1, torch.int64)
        self.glog = []
        self.exchange_log = []  # per batch: rows / bytes this rank sent per exchanged layer
        X = features if isinstance(features, torch.Tensor) else torch.as_tensor(np.asarray(features))
        X = X.to(dev, torch.float32)
        if X.shape[0] == n and n != self.n_own:
            X = X[r::P]
        if X.shape[0] != self.n_own:
            raise E.ShapeError(f"features rows {X.shape[0]}: expected {n} (global) or {self.n_own} (owned)")
        Xl = torch.zeros(cap, X.shape[1], dtype=torch.float32, device=dev)
        Xl[: self.n_own] = X
        self._gb = None
        super().__init__(bundle, g, Xl, max_batch=max_batch, update=update, bootstrap=False, use_graphs=False)
        self._refresh_ghosts([0])
        if bootstrap:
            self.bootstrap()

    # ---------------------------------------------------------------- plumbing
    def _cap_for(self, n_loc: int, B: int) -> int:
        h = self.ghost_headroom
        return int(min(self.n_glob, n_loc + max(int(h * n_loc), 4 * B if h > 0 else B, 64)))

    @property
    def cap(self) -> int:
        return self.g.n

    def _shard(self) -> _lib.Shard:
        p = _lib.ptr
        return _lib.Shard(self.comm.rank, self.comm.world, self.n_glob, self.n_own, self.g.n, p(self.g2l),
                          p(self.l2g), p(self.n_loc_t), p(self.peers), p(self.gout), p(self.gout_prev))

    def _mg(self) -> _lib.Graph:
        """Graph struct for the model kernels: shard adjacency + GLOBAL out-degrees."""
        g = self.g.c()
        g.out_deg, g.out_deg_prev = _lib.ptr(self.gout), _lib.ptr(self.gout_prev)
        return g

    def _rows_owned(self) -> int:
        return self.n_own

    def _ensure_ws(self, B):
        # the [n, d] δ region only when δ is not kept in self.delta (non-fused sum aggregators)
        ws_fn = (self.lib.rtec_workspace_bytes if (not getattr(self, "fused", False) and self.b.model in SUM_MODELS)
                 else self.lib.rtec_workspace_bytes_ext)
        need = int(ws_fn(self.n, max(int(B), 1), max(self.g.out.slots, self.g.inn.slots), self.max_dim))
        # batch validation / ghost admission scan over the global id space
        need = max(need, int(self.lib.rtec_build_workspace_bytes(self.n_glob, max(int(B), 1))))
        if self.g.ws.numel() < need:
            self.g.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)

    def _state(self, l, incremental: bool = False):
        s = super()._state(l, incremental)
        if l > 0:
            s.log_in = _lib.ptr(self.glog[l - 1]) if len(self.glog) >= l else None
        return s

    def _chg_buffers(self, l):
        f = self.fr[l]
        if f.bm_chg is None:
            f.bm_chg = torch.zeros(max((self.n + 31) // 32, 1), dtype=torch.int32, device=self.dev)
            f.chg_slot = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)
            f.chg_list = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)
            f.n_chg = torch.zeros(1, dtype=torch.int64, device=self.dev)
        while len(self.glog) <= l:
            self.glog.append(torch.zeros(0, dtype=torch.float32, device=self.dev))
        return f

    def _announce(self, g: DynamicGraph) -> None:
        """Load time: every ghost u tells owner(u) that this rank holds it, with its local
        out-degree here; owners set peers[] and sum the global out-degrees."""
        P, dev = self.comm.world, self.g2l.device
        lg = self.l2g[self.n_own:self.n_loc].to(torch.int64)
        deg = g.out_deg[self.n_own:self.n_loc].to(torch.int64)
        own = owner_of(lg, P)
        order = torch.argsort(own, stable=True)
        lg, deg, own = lg[order], deg[order], own[order]
        sc = torch.bincount(own, minlength=P).to(torch.int64)
        rc = self.comm.all_to_all_counts(sc)
        scl, rcl = sc.cpu().tolist(), rc.cpu().tolist()
        got = self.comm.all_to_all_rows(torch.stack([lg, deg], 1), scl, rcl)
        if got.numel() and self.n_own:
            li = got[:, 0] // P
            self.gout.index_add_(0, li, got[:, 1].to(torch.int32))
            src_rank = torch.repeat_interleave(torch.arange(P, device=dev), torch.as_tensor(rcl, device=dev))
            bits = torch.zeros(self.n_own, dtype=torch.int64, device=dev)  # unique (u, rank) pairs: sum == OR
            bits.index_add_(0, li, torch.ones_like(li) << src_rank)
            self.peers[: self.n_own] = bits.to(torch.int32)

    def _mats(self, layers):
        """(device pointers, widths) of the layer inputs H^l for l in `layers`."""
        return [self.H[l].data_ptr() for l in layers], [int(self.H[l].shape[1]) for l in layers]

    def _send_recv(self, peer_count: torch.Tensor, extra=None):
        """Per-peer send counts (device) -> (send counts, recv counts) on the host in one
        sync; `extra` device int64 scalars ride along in the same copy."""
        rc = self.comm.all_to_all_counts(peer_count)
        parts = [peer_count, rc] + ([t.reshape(-1) for t in extra] if extra else [])
        h = torch.cat(parts).cpu().numpy()
        P = self.comm.world
        return h[:P], h[P:2 * P], h[2 * P:]

    def _exchange_rows(self, mats, dims, send_counts, recv_counts, *, list_=None, n_list=None, max_list=0,
                       pair_u=None, pair_q=None, n_pairs=0, with_deg=False):
        """Pack (list or pair mode), all-to-all; returns the received (ids, degs, rows)."""
        P, dev = self.comm.world, self.dev
        k = int(np.sum(send_counts))
        off = np.zeros(P + 1, np.int64)
        off[1:] = np.cumsum(send_counts)
        ids = torch.zeros(max(k, 1), dtype=torch.int32, device=dev)
        deg = torch.zeros(max(k, 1), dtype=torch.int32, device=dev) if with_deg else None
        rows = torch.zeros(max(k, 1), sum(dims), dtype=torch.float32, device=dev)
        cursor = torch.zeros(P, dtype=torch.int64, device=dev)
        if k:
            p = _lib.ptr
            ma, mp = _ptr_array(mats)
            da, dp = _int_array(dims)
            oa, opp = _int_array(off, C.c_int64)
            _lib.check(self.lib.rtec_shard_pack(C.byref(self._shard()), len(mats), mp, dp, opp, p(list_), p(n_list),
                                                max_list, p(pair_u), p(pair_q), n_pairs, p(cursor), p(ids), p(deg),
                                                p(rows), _lib.stream_handle()), "shard_pack")
            del ma, da, oa
        r_ids = self.comm.all_to_all_rows(ids, send_counts, recv_counts)
        r_deg = self.comm.all_to_all_rows(deg, send_counts, recv_counts) if with_deg else None
        r_rows = self.comm.all_to_all_rows(rows, send_counts, recv_counts)
        return r_ids, r_deg, r_rows

    def _unpack_rows(self, mats, dims, ids, deg, rows, k, out_local=None):
        if not k:
            return
        ma, mp = _ptr_array(mats)
        da, dp = _int_array(dims)
        p = _lib.ptr
        _lib.check(self.lib.rtec_shard_unpack_rows(C.byref(self._shard()), len(mats), mp, dp, p(ids), p(deg),
                                                   p(rows), k, p(out_local), _lib.stream_handle()), "shard_unpack")
        del ma, da

    def _refresh_ghosts(self, layers):
        """Owners push the rows H^l (l in layers) of their owned vertices (chunked) to every
        rank holding a ghost of them, with the global out-degrees."""
        mats, dims = self._mats(layers)
        p, st = _lib.ptr, _lib.stream_handle()
        pc = torch.zeros(self.comm.world, dtype=torch.int64, device=self.dev)
        step = max(1, self.exchange_chunk)
        longest = int(self.comm.all_gather_ints([self.n_own], self.dev)[:, 0].max(initial=0))
        for c0 in range(0, max(longest, 1), step):
            cnt = max(min(step, self.n_own - c0), 0)
            lst = torch.arange(c0, c0 + cnt, dtype=torch.int32, device=self.dev)
            _lib.check(self.lib.rtec_shard_count_peers(C.byref(self._shard()), p(lst), None, cnt, p(pc), st),
                       "count_peers")
            sc, rc, _ = self._send_recv(pc)
            ids, deg, rows = self._exchange_rows(mats, dims, sc, rc, list_=lst, max_list=cnt, with_deg=True)
            self._unpack_rows(mats, dims, ids, deg, rows, int(np.sum(rc)))
        self.gout_prev.copy_(self.gout)

    # ---------------------------------------------------------------- bootstrap
    def bootstrap(self, sync: bool = True):
        """Full forward (models.py:461-477) of the owned rows over this rank's shard; after
        each layer the owners refresh the ghost rows of its output."""
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        st = _lib.stream_handle()
        p = _lib.ptr
        if getattr(self, "_own_ids", None) is None:
            self._own_ids = torch.arange(max(self.n_own, 1), dtype=torch.int32, device=self.dev)
            self._n_own_t = torch.tensor([self.n_own], dtype=torch.int64, device=self.dev)
        for l in range(self.L):
            g = self._mg()
            s = self._state(l)
            if self.b.model == GAT:  # Z / el / er of every local row feed the owned rows' softmax
                self._project(l, self.H[l], None, None, self.Z[l], self.el[l], self.er[l])
            # the owned rows only (local ids [0, n_own)): S / ctx / the final H hold n_own rows
            _lib.check(self.lib.rtec_layer_full(C.byref(g), C.byref(self.layers[l]), C.byref(s), p(self._own_ids),
                                                p(self._n_own_t), self.n_own, p(err), p(self.g.ws), self.g.ws.numel(),
                                                st), "bootstrap")
            if l + 1 < self.L:
                self._refresh_ghosts([l + 1])
        if sync:
            _lib.raise_err(err.item(), "bootstrap")

    run_full = bootstrap

    def refresh_projection(self, l: int) -> None:
        if self.b.model == GAT:
            self._project(l, self.H[l], None, None, self.Z[l], self.el[l], self.er[l])

    # ---------------------------------------------------------------- growth
    def _grow(self, need: int) -> None:
        """Local id capacity too small for a batch's possible admissions: rebuild the shard
        graph and every per-vertex array at a larger capacity (local ids are kept)."""
        new = self._cap_for(max(need, int(self.cap * 1.5)), 0)
        if new <= self.cap:
            return
        old = self.cap
        gr = self.g
        m = gr.num_edges
        v = torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)
        w = torch.empty_like(v)
        t = torch.empty(max(m, 1), dtype=torch.int64, device=self.dev)
        a = gr.out.c()
        ws = torch.empty(int(self.lib.rtec_build_workspace_bytes(old, max(m, 1))), dtype=torch.uint8, device=self.dev)
        _lib.check(self.lib.rtec_adj_export(old, C.byref(a), _lib.ptr(v), _lib.ptr(w), _lib.ptr(t), _lib.ptr(ws),
                                            ws.numel(), _lib.stream_handle()), "grow")
        self.g = DynamicGraph.from_tensors(new, v[:m], w[:m], t[:m], device=self.dev, reserve=self._reserve)

        def pad(x):
            if x is None:
                return None
            y = torch.zeros((new,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
            y[:old] = x[:old]
            return y

        for l in range(self.L):
            self.H[l] = pad(self.H[l])
        for lst in (self.Z, self.el, self.er, self.Zlog, self.erlog):
            for l in range(self.L):
                lst[l] = pad(lst[l])
        self.l2g = torch.cat([self.l2g, torch.full((new - old,), -1, dtype=torch.int32, device=self.dev)])
        self.gout, self.gout_prev = pad(self.gout), pad(self.gout_prev)
        self.dg_bm = torch.zeros(max((new + 31) // 32, 1), dtype=torch.int32, device=self.dev)
        if self.tc and self.b.model == GAT:
            pw = (max(self.b.dims[:-1]) + 31) // 32 * 32
            self.gemm_in = torch.zeros((new + 127) // 128 * 128 * pw, dtype=torch.float32, device=self.dev)
        self.n = new
        self.fr = [_Frontier(new, self.dev) for _ in range(self.L)]
        self.grown = getattr(self, "grown", 0) + 1
        self._ensure_ws(self.g.batch.cap)

    # ---------------------------------------------------------------- incremental step
    def enqueue_step(self, B: int) -> None:
        raise E.ConfigError("sharded engines synchronise inside a batch; use step()")

    def _global_batch(self, B: int):
        gb = self._gb
        if gb is None or gb["cap"] < max(B, 1):
            cap = max(B, 2 * (gb["cap"] if gb else 0), 1024)

            def z(dt, k=cap):
                return torch.zeros(k, dtype=dt, device=self.dev)

            gb = self._gb = {"cap": cap, "src": z(torch.int32), "dst": z(torch.int32), "op": z(torch.uint8),
                             "ts": z(torch.int64), "err": z(torch.int64, 1), "lsrc": z(torch.int32),
                             "ldst": z(torch.int32), "lop": z(torch.uint8), "lts": z(torch.int64),
                             "lpos": z(torch.int32), "nl": z(torch.int64, 1), "adm": z(torch.int32),
                             "n_adm": z(torch.int64, 1), "su": z(torch.int32), "sq": z(torch.int32),
                             "n_send": z(torch.int64, 1), "pc": z(torch.int64, self.comm.world),
                             "gst": z(torch.uint8)}
            self.sdelta = [z(torch.int32, 2 * cap) for _ in range(5)]
        return gb

    def _apply_local(self, B: int) -> None:
        gr = self.g
        for attempt in range(4):
            gr.apply_staged(B, phase=1)
            mine = gr.batch_error()
            word = combine_err_words(self.comm.all_gather_ints([_signed(mine)], self.dev)[:, 0])
            d = _lib.decode_err(word)
            if d is not None and d[0] == _lib.ARENA_FULL:
                # nothing mutated on any rank; ranks whose arena is short compact, all replay
                if _lib.decode_err(mine) is not None:
                    gr.compact(min_reserve=(16 * B + 4096) * 4 ** attempt)
                    gr._ensure_ws(gr.batch.cap, grow=2.0 ** (attempt + 1))
                    self._ensure_ws(gr.batch.cap)
                continue
            _lib.raise_err(word, "run_incremental", gr._ERR_MSG)
            gr.apply_staged(B, phase=2)
            return
        raise E.NativeError("run_incremental: arena still full after compaction")

    def step(self, op, src, dst, ts) -> RunResult:
        t0 = time.perf_counter()
        lib, st, p = self.lib, _lib.stream_handle(), _lib.ptr
        B = int(len(src))
        if self.n_loc + B > self.cap:  # room for every admission this batch could make
            self._grow(self.n_loc + B)
        gb = self._global_batch(B)
        for key, arr, dt in (("op", op, np.uint8), ("src", src, np.int32), ("dst", dst, np.int32),
                             ("ts", ts, np.int64)):
            if B:
                a = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(arr, dt)))
                gb[key][:B].copy_(a.to(gb[key].dtype), non_blocking=True)
        self._ensure_ws(max(B, self.g.batch.cap))
        ws, wsb = p(self.g.ws), self.g.ws.numel()
        sh = self._shard()
        # 1. validate (whole batch, every rank), admit ghosts, the shard's part of the batch
        _lib.check(lib.rtec_batch_validate(p(gb["src"]), p(gb["dst"]), B, self.n_glob, p(gb["err"]), ws, wsb, st),
                   "validate")
        _lib.check(lib.rtec_shard_admit(C.byref(sh), p(gb["src"]), p(gb["dst"]), p(gb["op"]), B, p(gb["err"]),
                                        p(self.bm_adm), p(gb["adm"]), p(gb["n_adm"]), p(gb["su"]), p(gb["sq"]),
                                        p(gb["n_send"]), p(gb["pc"]), ws, wsb, st), "admit")
        _lib.check(lib.rtec_shard_localize(C.byref(sh), p(gb["src"]), p(gb["dst"]), p(gb["op"]), p(gb["ts"]), B,
                                           p(gb["err"]), p(gb["lsrc"]), p(gb["ldst"]), p(gb["lop"]), p(gb["lts"]),
                                           p(gb["lpos"]), p(gb["nl"]), ws, wsb, st), "localize")
        sc, rc, ex = self._send_recv(gb["pc"], [gb["err"], gb["n_adm"], gb["nl"], gb["n_send"]])
        _lib.raise_err(int(ex[0]) & _U64, "run_incremental", self.g._ERR_MSG)  # identical on every rank
        n_adm, nl, n_send = int(ex[1]), int(ex[2]), int(ex[3])
        # 2. ghost admission: owners ship the new ghosts' pre-batch rows and out-degrees
        mats, dims = self._mats(range(self.L))
        ids, deg, rows = self._exchange_rows(mats, dims, sc, rc, pair_u=gb["su"], pair_q=gb["sq"], n_pairs=n_send,
                                             with_deg=True)
        k = int(np.sum(rc))
        if k:
            loc = torch.zeros(k, dtype=torch.int32, device=self.dev)
            self._unpack_rows(mats, dims, ids, deg, rows, k, loc)
            if self.b.model == GAT:
                nk = torch.tensor([k], dtype=torch.int64, device=self.dev)
                for l in range(self.L):
                    self._project(l, self.H[l], loc, nk, self.Z[l], self.el[l], self.er[l])
        self.n_loc += n_adm
        self.admitted = n_adm
        # 3. apply the shard's updates (two phases, status words combined in between)
        gr = self.g
        gr.stage(gb["lop"][:nl], gb["lsrc"][:nl], gb["ldst"][:nl], gb["lts"][:nl])
        self._ensure_ws(gr.batch.cap)
        ws, wsb = p(gr.ws), gr.ws.numel()
        self._apply_local(nl)
        bb = gr.batch
        gst = gb["gst"][: max(B, 1)]
        gst.zero_()
        if nl:
            gst.index_copy_(0, gb["lpos"][:nl].to(torch.int64), bb.status[:nl])
        self.comm.all_reduce_(gst, op=dist.ReduceOp.MAX)
        sd = self.sdelta
        _lib.check(lib.rtec_shard_degrees(C.byref(sh), p(gb["src"]), p(gb["dst"]), p(gb["op"]), p(gst), B,
                                          p(gr.in_deg), p(gr.in_deg_prev), p(self.bm_touch), p(self.dg_bm), p(sd[0]),
                                          p(sd[1]), p(sd[2]), p(sd[3]), p(sd[4]), p(self.n_sdelta), ws, wsb, st),
                   "shard_degrees")
        # 4. layers, one targeted exchange after each but the last
        g = self._mg()
        b = bb.c()
        b.dg_bm = p(self.dg_bm)
        sdd = 1 if self.b.src_degree_dependent else 0
        fc = [None] * self.L
        self.exchange_log.append([])
        for l in range(self.L):
            prev = C.byref(fc[l - 1]) if l > 0 else None
            fc[l] = self.fr[l].c()
            _lib.check(lib.rtec_frontier_layer(C.byref(g), C.byref(b), l, sdd, prev, C.byref(fc[l]), ws, wsb, st),
                       "frontier")
            if self.b.model == GAT and l > 0:
                pf = self.fr[l - 1]
                _lib.check(lib.rtec_gat_project(C.byref(self.layers[l]), p(self.H[l]), p(pf.chg_list), p(pf.n_chg),
                                                self.n, p(self.Z[l]), p(self.el[l]), p(self.er[l]), p(self.Zlog[l]),
                                                p(self.erlog[l]), p(bb.err), self._proj_img(), st), "gat_project")
            s = self._state(l, incremental=True)
            _lib.check(lib.rtec_layer_incremental(C.byref(g), C.byref(b), C.byref(self.layers[l]), C.byref(s), prev,
                                                  C.byref(fc[l]), p(bb.err), ws, wsb, st), "layer")
            if l + 1 < self.L:
                self._exchange_layer(l)
                fc[l] = self.fr[l].c()  # now carries bm_chg / chg_slot
        # 5. close the batch
        mine = gr.batch_error()
        word = combine_err_words(self.comm.all_gather_ints([_signed(mine)], self.dev)[:, 0])
        _lib.raise_err(word, "run_incremental", gr._ERR_MSG)
        _lib.check(lib.rtec_batch_commit(C.byref(gr.c()), C.byref(bb.c()), st), "commit")
        _lib.check(lib.rtec_shard_commit(C.byref(sh), p(gb["src"]), p(gb["dst"]), p(gst), B, p(self.dg_bm),
                                         p(self.bm_touch), st), "shard_commit")
        status = gst[:B].cpu().numpy().copy()
        kd = int(self.n_sdelta.item())
        rows_d = self.comm.all_gather_var(torch.stack([t[: max(kd, 1)] for t in sd], 1), kd)
        dd = rows_d.cpu().numpy().astype(np.int64)
        deltas = dd[np.argsort(dd[:, 0], kind="stable")] if len(dd) else np.zeros((0, 5), np.int64)
        m = self.metrics()
        m.wall_time = time.perf_counter() - t0
        return RunResult(status, deltas, None, m)

    def _exchange_layer(self, l: int) -> None:
        """Targeted exchange of layer l's changed owned rows (H^{l+1}) to the ranks holding
        ghosts of them, in rounds of at most `exchange_chunk` listed rows per rank (bounded
        send / receive buffers); assembles V_chg(l) and, for the next layer, either the
        received rows' source deltas (fused sum aggregators) or the exchanged DeltaLog."""
        lib, st, p = self.lib, _lib.stream_handle(), _lib.ptr
        f = self._chg_buffers(l)
        H = self.H[l + 1]
        d = int(H.shape[1])
        fused = self.fused
        pc = torch.zeros(self.comm.world, dtype=torch.int64, device=self.dev)
        n_dst = int(f.n_dst.item())
        rounds = int(self.comm.all_gather_ints([n_dst], self.dev)[:, 0].max(initial=0))
        step = max(1, self.exchange_chunk)
        rounds = max((rounds + step - 1) // step, 1)
        sent = recv = 0
        for rd in range(rounds):
            c0 = min(rd * step, n_dst)
            cnt = max(min(step, n_dst - c0), 0)
            lst = f.dst_list[c0:c0 + cnt] if cnt else f.dst_list[:1]
            _lib.check(lib.rtec_shard_count_peers(C.byref(self._shard()), p(lst), None, cnt, p(pc), st), "count_peers")
            sc, rc, _ = self._send_recv(pc)
            ids, _, rows = self._exchange_rows([H.data_ptr()], [d], sc, rc, list_=lst, max_list=cnt)
            k = int(np.sum(rc))
            last = rd == rounds - 1
            if not fused:
                need = max(recv + k + (n_dst if last else 0), 1) * d
                if self.glog[l].numel() < need:  # grow, keeping the rows of earlier rounds
                    g2 = torch.zeros(int(need * 1.25), dtype=torch.float32, device=self.dev)
                    g2[: self.glog[l].numel()] = self.glog[l]
                    self.glog[l] = g2
            _lib.check(lib.rtec_shard_unpack_changed(
                C.byref(self._shard()), d, p(ids), p(rows), k, recv, 1 if rd == 0 else 0, p(H),
                p(f.dst_list) if last else None, p(f.n_dst), n_dst, p(self.log[l]), p(f.dst_slot),
                None if fused else p(self.glog[l]), p(self.delta[l + 1]) if fused else None,
                1 if self.b.model == GCN else 0, float(self.b.degree_offset), p(f.bm_chg), p(f.chg_slot),
                p(f.chg_list), p(f.n_chg), st), "shard_unpack")
            sent += int(np.sum(sc))
            recv += k
        self.exchange_log[-1].append({"layer": l, "rounds": rounds, "rows_sent": sent, "rows_recv": recv,
                                      "bytes_sent": sent * (4 * d + 4)})

    # ---------------------------------------------------------------- reads
    def _owned_popcount(self, bm: torch.Tensor) -> int:
        words = bm[: (self.n_own + 31) // 32].to(torch.int64) & 0xFFFFFFFF
        if self.n_own % 32 and words.numel():
            words[-1] &= (1 << (self.n_own % 32)) - 1
        c = torch.zeros_like(words)
        for b in range(32):
            c += (words >> b) & 1
        return int(c.sum().item())

    def metrics(self) -> Metrics:
        """Counters summed over ranks (|E_curr|, |V_dst|, Σindeg; |S| counted at the owners)."""
        m = Metrics()
        for f in self.fr:
            c = f.counters.clone()
            c[2] = self._owned_popcount(f.bm_src)
            self.comm.all_reduce_(c)
            c = c.cpu().numpy()
            m.e_curr.append(int(c[0]))
            m.v_dst.append(int(c[1]))
            m.n_src.append(int(c[2]))
            m.in_edges_vdst.append(int(c[5]))
        m.as_edges, m.as_vertices = sum(m.e_curr), sum(m.v_dst)
        return m

    def embeddings(self, l: int) -> np.ndarray:
        """Full H^l assembled from the owners' rows (collective)."""
        d = self.H[l].shape[1]
        full = torch.zeros(self.n_glob, d, dtype=torch.float32, device=self.dev)
        full[self.l2g[: self.n_own].to(torch.int64)] = self.H[l][: self.n_own]
        self.comm.all_reduce_(full)
        return full.cpu().numpy()

    def frontier(self, l: int):
        """(V_dst(l), S(l)) over all ranks, ascending global ids (collective)."""
        f = self.fr[l]
        nd = int(f.n_dst.item())
        vd = self.l2g[f.dst_list[:nd].to(torch.int64)]
        vd = self.comm.all_gather_var(vd, nd)
        ns = int(f.n_src.item())
        sl = f.src_list[:ns].to(torch.int64)
        so = self.l2g[sl[sl < self.n_own]]
        so = self.comm.all_gather_var(so, int(so.numel()))
        return np.sort(vd.cpu().numpy().astype(np.int64)), np.sort(so.cpu().numpy().astype(np.int64))

    def query(self, ids) -> np.ndarray:
        """Final-layer rows for `ids`, each read on its owner (collective)."""
        ids_np = np.asarray(ids, np.int64)
        if ids_np.size and (ids_np.min() < 0 or ids_np.max() >= self.n_glob):
            raise E.InvalidVertex("query vertex outside the vertex range")
        ids_t = torch.as_tensor(ids_np, device=self.dev)
        P = self.comm.world
        mine = owner_of(ids_t, P) == self.comm.rank
        out = torch.zeros(ids_np.size, self.b.dims[-1], dtype=torch.float32, device=self.dev)
        if ids_np.size:
            out[mine] = self.H[-1][ids_t[mine] // P]  # owned rows at local v // P
        self.comm.all_reduce_(out)
        return out.cpu().numpy()

    materialize_h = query

    def memory_bytes(self) -> dict:
        """HBM held by this rank's shard, by class (the replica-free store)."""
        def nb(xs):
            return sum(x.numel() * x.element_size() for x in xs if x is not None)

        gr = self.g
        return {"n_own": self.n_own, "n_local": self.n_loc, "cap": self.cap,
                "layer_inputs": nb(self.H[: self.L]),
                "owned_state": nb([self.H[self.L]] + self.S + self.ctx + self.log),
                "gat_caches": nb(self.Z + self.el + self.er + self.Zlog + self.erlog),
                "source_deltas": self.delta[0].untyped_storage().nbytes() if self.fused else 0,
                "exchanged_log": nb(self.glog),
                "graph": nb([gr.out.nbr, gr.out.ts, gr.inn.nbr, gr.out.beg, gr.inn.beg, gr.out.len, gr.inn.len,
                             gr.out.cap, gr.inn.cap]),
                "maps": nb([self.g2l, self.l2g, self.peers, self.gout, self.gout_prev]),
                "workspace": gr.ws.numel()}

    def shard_edges(self):
        """This rank's edges (src, dst, ts) in global ids."""
        s, d, t = self.g.edges()
        l2g = self.l2g.cpu().numpy().astype(np.int64)
        return l2g[s], l2g[d], t

    def save(self, directory: str) -> None:
        """Per-rank checkpoint (formats.save_sharded_checkpoint); call on every rank."""
        from .formats import save_sharded_checkpoint

        save_sharded_checkpoint(self, directory)

    @staticmethod
    def load(directory: str, comm: Comm | None = None, **kw) -> "ShardedRTECEngine":
        """Resume this rank's shard (formats.load_sharded_checkpoint); collective."""
        from .formats import load_sharded_checkpoint

        return load_sharded_checkpoint(directory, comm if comm is not None else Comm(), **kw)

    def aggregates(self, l: int):
        raise E.ConfigError("aggregates() of a sharded engine: read owned rows of S[l] on each rank")
