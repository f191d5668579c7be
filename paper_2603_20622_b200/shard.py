"""Vertex-sharded incremental engine: one process per GPU.

The reference is single-process CPU code; the paper offloads
historical embeddings to host memory.  Here they are
sharded over the GPUs' HBM instead:

- owner(v) = v mod P.  Rank p's `DynamicGraph` shard holds every edge whose
  dst it owns, in both directions (in-runs for aggregation, out-runs for
  frontier expansion).  `rtec_batch_apply_phase` validates the WHOLE batch on
  every rank (so errors are identical everywhere and raised before any shard
  mutates) and probes / merges only owned-dst updates.
- Out-degrees are global (GCN's 1/sqrt(d_out(u)+off), models.py:98-99, and
  the F1 frontier's Dg seed): every rank keeps replicated global degree
  arrays, updated by `rtec_shard_degrees` from the globally applied set
  (per-update status MAX-all-reduced over ranks; each update has exactly one
  owner).
- Every layer input H^0..H^{L-1} is replicated; after layer l computes its
  owned changed rows V_dst(l), one halo exchange per layer (all-gather of
  (id, row) over NCCL) refreshes the replicas and assembles V_chg(l) and the
  exchanged DeltaLog (pre-batch rows) that layer l+1 reads.  No exchange is
  needed after the last layer; `query` gathers rows from their owners.

Collectives go through `Comm`: device tensors over NCCL (NVLink/NVSwitch);
with a gloo group (CPU tests, or ranks sharing one GPU) tensors are staged
through host memory.  The per-batch host synchronisations are the error-word
combine between apply's plan and mutate phases and the row counts of each
exchange.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import errors as E
from .engine import Metrics, RTECEngine, RunResult
from .graph import DynamicGraph
from .models import GAT, PROJECTED

_U64 = (1 << 64) - 1


def owner_of(v, world: int):
    """Partition function of the shards (== rtec_graph_t part_rank / part_count)."""
    return v % world


class Comm:
    """The four collectives the sharded engine issues, over torch.distributed."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = str(dist.get_backend(group))
        self.staged = self.backend != "nccl"

    def _dev(self, like: torch.Tensor):
        return torch.device("cpu") if self.staged else like.device

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

    def all_gather_rows(self, ids: torch.Tensor, rows: torch.Tensor):
        """Every rank's equally sized (ids [cap], rows [cap, d]) -> ([world*cap], [world*cap, d])."""
        dev = ids.device
        if self.staged:
            i_h, r_h = ids.cpu(), rows.cpu()
            gi = [torch.empty_like(i_h) for _ in range(self.world)]
            gr = [torch.empty_like(r_h) for _ in range(self.world)]
            dist.all_gather(gi, i_h, group=self.group)
            dist.all_gather(gr, r_h, group=self.group)
            return torch.cat(gi).to(dev), torch.cat(gr).to(dev)
        out_i = torch.empty(self.world * ids.numel(), dtype=ids.dtype, device=dev)
        out_r = torch.empty((self.world * rows.shape[0],) + tuple(rows.shape[1:]), dtype=rows.dtype, device=dev)
        dist.all_gather_into_tensor(out_i, ids.contiguous(), group=self.group)
        dist.all_gather_into_tensor(out_r, rows.contiguous(), group=self.group)
        return out_i, out_r


def combine_err_words(words) -> int:
    """Status words of all ranks -> the batch's word: smallest (position, code) wins (unsigned)."""
    return min(int(w) & _U64 for w in words)


class ShardedRTECEngine(RTECEngine):
    """RTECEngine over this rank's shard; same step()/query() API."""

    FUSED_DELTA = False  # the halo exchange ships new rows and rebuilds the DeltaLog on receipt

    def __init__(self, bundle, num_vertices: int, edges, features, comm: Comm, *, max_batch: int | None = None,
                 update: str = "tc", reserve: int | None = None, device=None, exchange_chunk: int = 1 << 20,
                 bootstrap: bool = True):
        if bundle.model in PROJECTED:  # payload / gate caches are not exchanged between shards
            raise E.UnsupportedModel(f"sharded engine: model {bundle.model!r} not supported")
        self.comm = comm
        P, r = comm.world, comm.rank
        n = int(num_vertices)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        src, dst = (torch.as_tensor(np.asarray(a) if not isinstance(a, torch.Tensor) else a, device=dev)
                    for a in edges[:2])
        ts = edges[2] if len(edges) > 2 else None
        ts = (torch.arange(src.numel(), dtype=torch.int64, device=dev) if ts is None
              else torch.as_tensor(np.asarray(ts) if not isinstance(ts, torch.Tensor) else ts, device=dev))
        mine = owner_of(dst.to(torch.int64), P) == r
        g = DynamicGraph.from_tensors(n, src[mine], dst[mine], ts[mine], device=dev,
                                      reserve=reserve if reserve is not None else None)
        g.part_rank, g.part_count = r, P
        self.exchange_chunk = int(exchange_chunk)
        words = (n + 31) // 32
        # replicated global degrees (local out-degrees sum to the global one; in-degrees live on the owner)
        self.gout = comm.all_reduce_(g.out_deg.clone())
        self.gin = comm.all_reduce_(g.in_deg.clone())
        self.gout_prev, self.gin_prev = self.gout.clone(), self.gin.clone()
        zi = lambda k, dt=torch.int32: torch.zeros(max(k, 1), dtype=dt, device=dev)  # noqa: E731
        self.bm_touch, self.dg_bm = zi(words), zi(words)
        self.gdelta = [zi(2 * (max_batch or g.batch.cap)) for _ in range(5)]
        self.n_gdelta = zi(1, torch.int64)
        self.gstatus = torch.zeros(max(max_batch or 1, 1), dtype=torch.uint8, device=dev)
        self.owned = torch.arange(r, n, P, dtype=torch.int32, device=dev)
        self.n_owned = torch.tensor([self.owned.numel()], dtype=torch.int64, device=dev)
        self.glog = []  # per exchanged layer: DeltaLog rows of V_chg(l) in exchange order
        super().__init__(bundle, g, features, max_batch=max_batch, update=update, bootstrap=bootstrap)

    # ---------------------------------------------------------------- plumbing
    def _mg(self) -> _lib.Graph:
        """Graph struct for the model kernels: shard adjacency + GLOBAL out-degrees."""
        g = self.g.c()
        g.out_deg, g.out_deg_prev = _lib.ptr(self.gout), _lib.ptr(self.gout_prev)
        return g

    def _rows_owned(self) -> int:
        # owner(v) = v mod P: rank r owns r, r + P, ...; its rows sit at v // P
        P, r = self.comm.world, self.comm.rank
        return max((self.n - r + P - 1) // P, 0)

    def _ensure_ws(self, B):
        # the δ rows live in per-layer buffers sized |S(l)| (slot-indexed), not in the workspace
        need = int(self.lib.rtec_workspace_bytes_ext(self.n, max(int(B), 1),
                                                     max(self.g.out.slots, self.g.inn.slots), self.max_dim))
        if self.g.ws.numel() < need:
            self.g.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)

    def _delta_buffer(self, l: int, rows: int) -> torch.Tensor:
        if not hasattr(self, "_dbuf"):
            self._dbuf = [torch.zeros(1, dtype=torch.float32, device=self.dev) for _ in range(self.L)]
        need = max(rows, 1) * int(self.b.agg_dims[l])
        if self._dbuf[l].numel() < need:
            self._dbuf[l] = torch.zeros(int(need * 1.25), dtype=torch.float32, device=self.dev)
        return self._dbuf[l]

    def _state(self, l, incremental: bool = False):
        s = super()._state(l, incremental)
        if l > 0:
            s.log_in = _lib.ptr(self.glog[l - 1]) if len(self.glog) >= l else None
        # destination-side rows per owned vertex (v // P); δ rows per S(l) slot
        s.row_div = self.comm.world
        s.out_local = 1 if l + 1 == self.L else 0
        s.delta_slot = 1
        return s

    def _chg_buffers(self, l):
        f = self.fr[l]
        if f.bm_chg is None:
            words = (self.n + 31) // 32
            f.bm_chg = torch.zeros(max(words, 1), dtype=torch.int32, device=self.dev)
            f.chg_slot = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)
            f.chg_list = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)
            f.n_chg = torch.zeros(1, dtype=torch.int64, device=self.dev)
        while len(self.glog) <= l:
            self.glog.append(torch.zeros(0, dtype=torch.float32, device=self.dev))
        return f

    def _exchange(self, H: torch.Tensor, d: int, rows: torch.Tensor, count: int, *, layer: int | None = None):
        """All-gather (id, row) of this rank's `count` rows H[rows[:count]] and
        unpack them into the replica H.  With `layer`, also assemble V_chg(layer),
        chg_slot and the exchanged DeltaLog (pre-batch rows) for layer + 1."""
        lib, st, P = self.lib, _lib.stream_handle(), self.comm.world
        counts = self.comm.all_gather_ints([count], self.dev)[:, 0]
        mg = self.g.c()
        p = _lib.ptr
        if layer is None:  # replica refresh (bootstrap): chunked, positions irrelevant
            step = max(1, self.exchange_chunk)
            for c0 in range(0, int(counts.max(initial=0)), step):
                ck = np.clip(counts - c0, 0, step)
                cap = int(ck.max())
                mine = int(ck[self.comm.rank])
                ids = torch.zeros(cap, dtype=torch.int32, device=self.dev)
                buf = torch.zeros(cap, d, dtype=torch.float32, device=self.dev)
                if mine:
                    _lib.check(lib.rtec_halo_pack(p(H), d, p(rows[c0:]), None, mine, p(ids), p(buf), st), "halo_pack")
                rid, rrow = self.comm.all_gather_rows(ids, buf)
                cnt = torch.as_tensor(ck, dtype=torch.int64, device=self.dev)
                _lib.check(lib.rtec_halo_unpack(C.byref(mg), d, p(rid), p(rrow), p(cnt), P, cap, p(H), None, None, None,
                                                None, None, None, None, st), "halo_unpack")
            return
        f = self._chg_buffers(layer)
        total = int(counts.sum())
        cap = max(int(counts.max(initial=0)), 1)
        if self.glog[layer].numel() < max(total, 1) * d:
            self.glog[layer] = torch.zeros(max(total, 1) * d, dtype=torch.float32, device=self.dev)
        ids = torch.zeros(cap, dtype=torch.int32, device=self.dev)
        buf = torch.zeros(cap, d, dtype=torch.float32, device=self.dev)
        if count:
            _lib.check(lib.rtec_halo_pack(p(H), d, p(rows), None, count, p(ids), p(buf), st), "halo_pack")
        rid, rrow = self.comm.all_gather_rows(ids, buf)
        cnt = torch.as_tensor(counts, dtype=torch.int64, device=self.dev)
        loc = self.fr[layer]
        _lib.check(lib.rtec_halo_unpack(C.byref(mg), d, p(rid), p(rrow), p(cnt), P, cap, p(H), p(self.log[layer]),
                                        p(loc.dst_slot), p(self.glog[layer]), p(f.bm_chg), p(f.chg_slot),
                                        p(f.chg_list), p(f.n_chg), st), "halo_unpack")

    # ---------------------------------------------------------------- bootstrap
    def bootstrap(self, sync: bool = True):
        """Full forward (models.py:461-477) of the owned rows over this rank's shard,
        then the owners' rows refresh the replicas."""
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        st = _lib.stream_handle()
        p = _lib.ptr
        for l in range(self.L):
            g = self._mg()
            s = self._state(l)
            if self.b.model == GAT:  # Z / el / er of every (replica) row feed the owned rows' softmax
                _lib.check(self.lib.rtec_gat_project(C.byref(self.layers[l]), p(self.H[l]), None, None, self.n,
                                                     p(self.Z[l]), p(self.el[l]), p(self.er[l]), None, None, None,
                                                     self._proj_img(), st), "bootstrap")
            _lib.check(self.lib.rtec_layer_full(C.byref(g), C.byref(self.layers[l]), C.byref(s), p(self.owned),
                                                p(self.n_owned), self.owned.numel(), p(err), p(self.g.ws),
                                                self.g.ws.numel(), st), "bootstrap")
            if l + 1 < self.L:
                self._exchange(self.H[l + 1], self.b.dims[l + 1], self.owned, self.owned.numel())
        _lib.raise_err(err.item(), "bootstrap")

    run_full = bootstrap

    # ---------------------------------------------------------------- incremental step
    def enqueue_step(self, B: int) -> None:
        raise E.ConfigError("sharded engines synchronise inside a batch; use step()")

    def _apply(self, B: int) -> None:
        gr = self.g
        for attempt in range(4):
            gr.apply_staged(B, phase=1)
            mine = gr.batch_error()
            word = combine_err_words(self.comm.all_gather_ints([mine - (1 << 64) if mine >= (1 << 63) else mine],
                                                               self.dev)[:, 0])
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
        gr = self.g
        B = gr.stage(op, src, dst, ts)
        if self.gstatus.numel() < max(B, 1):
            self.gstatus = torch.zeros(gr.batch.cap, dtype=torch.uint8, device=self.dev)
            self.gdelta = [torch.zeros(2 * gr.batch.cap, dtype=torch.int32, device=self.dev) for _ in range(5)]
        self._ensure_ws(gr.batch.cap)
        self._apply(B)
        lib, st, p = self.lib, _lib.stream_handle(), _lib.ptr
        bb = gr.batch
        gst = self.gstatus[:max(B, 1)]
        gst.copy_(bb.status[:max(B, 1)])
        self.comm.all_reduce_(gst, op=dist.ReduceOp.MAX)
        gd = self.gdelta
        _lib.check(lib.rtec_shard_degrees(self.n, p(bb.src), p(bb.dst), p(bb.op), p(gst), B, p(self.gout),
                                          p(self.gout_prev), p(self.gin), p(self.gin_prev), p(self.bm_touch),
                                          p(self.dg_bm), p(gd[0]), p(gd[1]), p(gd[2]), p(gd[3]), p(gd[4]),
                                          p(self.n_gdelta), p(gr.ws), gr.ws.numel(), st), "shard_degrees")
        g = self._mg()
        b = bb.c()
        b.dg_bm = p(self.dg_bm)
        sdd = 1 if self.b.src_degree_dependent else 0
        ws, wsb = p(gr.ws), gr.ws.numel()
        fc = [None] * self.L
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
            s = self._state(l)
            s.delta = p(self._delta_buffer(l, int(self.fr[l].n_src.item())))  # |S(l)| δ rows
            _lib.check(lib.rtec_layer_incremental(C.byref(g), C.byref(b), C.byref(self.layers[l]), C.byref(s), prev,
                                                  C.byref(fc[l]), p(bb.err), ws, wsb, st), "layer")
            if l + 1 < self.L:
                cnt = int(self.fr[l].n_dst.item())
                self._exchange(self.H[l + 1], self.b.dims[l + 1], self.fr[l].dst_list, cnt, layer=l)
                fc[l] = self.fr[l].c()  # now carries bm_chg / chg_slot
        mine = gr.batch_error()
        word = combine_err_words(self.comm.all_gather_ints([mine - (1 << 64) if mine >= (1 << 63) else mine],
                                                           self.dev)[:, 0])
        _lib.raise_err(word, "run_incremental", gr._ERR_MSG)
        _lib.check(lib.rtec_batch_commit(C.byref(gr.c()), C.byref(bb.c()), st), "commit")
        _lib.check(lib.rtec_shard_commit(p(bb.src), p(bb.dst), p(gst), B, p(self.gout), p(self.gout_prev),
                                         p(self.gin), p(self.gin_prev), p(self.bm_touch), p(self.dg_bm), st),
                   "shard_commit")
        status = gst[:B].cpu().numpy().copy()
        k = int(self.n_gdelta.item())
        deltas = (np.stack([t[:k].cpu().numpy().astype(np.int64) for t in gd], axis=1) if k
                  else np.zeros((0, 5), np.int64))
        return RunResult(status, deltas, None, self.metrics())

    # ---------------------------------------------------------------- reads
    def metrics(self) -> Metrics:
        """Counters summed over ranks (|E_curr|, |V_dst|, Σindeg); |S| is global already."""
        m = Metrics()
        for f in self.fr:
            c = f.counters.clone()
            self.comm.all_reduce_(c)
            c = c.cpu().numpy()
            m.e_curr.append(int(c[0]))
            m.v_dst.append(int(c[1]))
            m.n_src.append(int(f.counters[2].item()))
            m.in_edges_vdst.append(int(c[5]))
        return m

    def owned_rows(self, t: torch.Tensor) -> torch.Tensor:
        return t[self.owned.to(torch.int64)]

    def embeddings(self, l: int) -> np.ndarray:
        """Full H^l assembled from the owners' rows (collective)."""
        d = self.H[l].shape[1]
        full = torch.zeros(self.n, d, dtype=torch.float32, device=self.dev)
        idx = self.owned.to(torch.int64)
        # the final layer is stored per owned vertex (row v // P); inputs are full replicas
        full[idx] = self.H[l][: idx.numel()] if l == self.L else self.H[l][idx]
        self.comm.all_reduce_(full)
        return full.cpu().numpy()

    def frontier(self, l: int):
        """(V_dst(l) over all ranks, S(l)) ascending (collective)."""
        f = self.fr[l]
        bm = f.bm_dst.clone()
        self.comm.all_reduce_(bm)  # shards' V_dst are disjoint: SUM == OR
        bits = ((bm.cpu().numpy().view(np.uint32)[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
        vd = np.flatnonzero(bits.reshape(-1))[: self.n]
        ns = int(f.n_src.item())
        return vd.astype(np.int64), f.src_list[:ns].cpu().numpy().astype(np.int64)

    def query(self, ids) -> np.ndarray:
        """Final-layer rows for `ids`, each read on its owner (collective)."""
        ids_np = np.asarray(ids, np.int64)
        if ids_np.size and (ids_np.min() < 0 or ids_np.max() >= self.n):
            raise E.InvalidVertex("query vertex outside the vertex range")
        ids_t = torch.as_tensor(ids_np, device=self.dev)
        P = self.comm.world
        mine = owner_of(ids_t, P) == self.comm.rank
        out = torch.zeros(ids_np.size, self.b.dims[-1], dtype=torch.float32, device=self.dev)
        if ids_np.size:
            out[mine] = self.H[-1][ids_t[mine] // P]  # owned rows at v // P
        self.comm.all_reduce_(out)
        return out.cpu().numpy()

    materialize_h = query

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
