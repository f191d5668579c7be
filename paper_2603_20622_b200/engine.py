"""Incremental RTEC engine on B200 (the SPEC engines/state_cache/frontier layer).

The reference ships no engine; this implements its
contract: `bootstrap` (== layer_embeddings per layer,
models.py:461-477), `run_incremental` (Alg. 1 / Alg. 3 on
the F1 frontier), `run_full`, `query` / `materialize_h`
(SPEC.md:379), with device-side access counters (SPEC.md:430-433 Metrics).

Per batch the host only enqueues C-ABI calls on one stream:

    rtec_batch_apply            graph.py:184 apply_batch (validate, probe, merge, deltas)
    for l in 0..L-1:
      rtec_frontier_layer       Alg. 4 layer l (F1 rule)
      rtec_gat_project          GAT only, l >= 1: Z/el/er of V_chg(l-1) rows (+ DeltaLog)
      rtec_layer_incremental    Alg. 1 / Alg. 3 + recompute R(l) + update GEMM (+ DeltaLog)
    rtec_batch_commit           degree snapshots catch up

No host synchronisation happens inside a batch (all sizes stay on the
device), so the whole step can be captured in a CUDA graph (`capture()`).
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import errors as E
from .graph import DynamicGraph, EdgeUpdate, updates_to_arrays
from .models import AGNN, COMMNET, GAT, GCN, GGCN, GIN, GIN_FAMILY, GIN_MAX, GRAPHSAGE, MONET, PINSAGE, Bundle, MODELS

_MODEL_ID = _lib.MODEL_IDS


@dataclass
class Metrics:
    """Per-layer device counters."""

    e_curr: list = field(default_factory=list)   # |E_curr(l)|
    v_dst: list = field(default_factory=list)    # |V_dst(l)|
    n_src: list = field(default_factory=list)    # |S(l)|
    in_edges_vdst: list = field(default_factory=list)  # Σ indeg(V_dst(l)) (scanned in-runs)
    mode: str = "inc"                            # inc | uer | full
    edge_accesses: list = field(default_factory=list)    # per layer, for `mode`
    vertex_accesses: list = field(default_factory=list)
    as_edges: int = 0                            # affected subgraph: Σ_l |E_curr(l)|
    as_vertices: int = 0                         # Σ_l |V_dst(l)|
    wall_time: float = 0.0                       # host seconds of the step, sync included
    refreshed: bool = False                      # refresh_every fired after this batch (full bootstrap)


def redundancy(m: Metrics, num_edges: int, num_vertices: int, breakdown: dict | None = None) -> dict:
    """SPEC cmd_redundancy_report: access volume of each strategy relative to
    the affected subgraph (Fig. 2 / Table V): FN = full-neighbour recompute of
    every layer, UER = affected rows over their full in-neighbourhoods, Inc = the incremental
    engine (exactly the affected edges); `redundant_share` = the part of FN's accesses outside
    the affected subgraph.  `breakdown` (RTECEngine.degree_breakdown) adds the per
    degree-class volumes."""
    L = len(m.e_curr)
    a = max(m.as_edges, 1)
    fn = L * int(num_edges)
    out = {"as_edges": m.as_edges, "as_vertices": m.as_vertices,
           "fn_edges": fn, "uer_edges": sum(m.in_edges_vdst), "inc_edges": sum(m.e_curr),
           "fn_over_as": fn / a, "uer_over_as": sum(m.in_edges_vdst) / a,
           "inc_over_as": sum(m.e_curr) / a, "fn_vertices": L * int(num_vertices),
           "redundant_share": (fn - m.as_edges) / fn if fn else 0.0}
    if breakdown is not None:
        out["degree_classes"] = breakdown
    return out


class RunResult:
    """status u8[B] (1 applied), deltas int32[k, 5] DegreeDelta rows, metrics, and
    `changed_final`: ascending ids of the vertices whose final-layer embedding was
    recomputed (inc / uer / ns: V_dst(L-1) of the batch; full: every vertex; odec: none,
    the rows are deferred).  The id list is snapshotted on the device at the end of the
    step and copied to the host on first access."""

    __slots__ = ("status", "deltas", "metrics", "_changed")

    def __init__(self, status, deltas, changed_final, metrics):
        self.status, self.deltas, self.metrics = status, deltas, metrics
        self._changed = changed_final

    @property
    def changed_final(self) -> np.ndarray:
        c = self._changed
        if isinstance(c, torch.Tensor):
            c = self._changed = c.cpu().numpy().astype(np.int64)
        return c


class _Frontier:
    def __init__(self, n, dev):
        words = (n + 31) // 32
        z = lambda k, dt: torch.zeros(max(k, 1), dtype=dt, device=dev)  # noqa: E731
        self.bm_src, self.bm_dst = z(words, torch.int32), z(words, torch.int32)
        self.src_list, self.dst_list = z(n, torch.int32), z(n, torch.int32)
        self.n_src, self.n_dst = z(1, torch.int64), z(1, torch.int64)
        self.src_slot, self.dst_slot = z(n, torch.int32), z(n, torch.int32)
        self.counters = z(8, torch.int64)
        # sharded runs (shard.py): V_chg(l) over all ranks + exchanged DeltaLog slots
        self.bm_chg = self.chg_slot = self.chg_list = self.n_chg = None

    def c(self):
        p = _lib.ptr
        return _lib.Frontier(p(self.bm_src), p(self.bm_dst), p(self.src_list), p(self.n_src), p(self.dst_list),
                             p(self.n_dst), p(self.src_slot), p(self.dst_slot), p(self.counters), p(self.bm_chg),
                             p(self.chg_slot))


class RTECEngine:
    """B200 incremental engine over a DynamicGraph and an operator Bundle."""

    FUSED_DELTA = True
    GAT_IMG_BUDGET = 8 << 30  # bytes of the GAT projection's tcgen05 A image (all n rows)

    def __init__(self, bundle: Bundle, graph: DynamicGraph, features, *, max_batch: int | None = None,
                 update: str = "tc", use_graphs: bool = True, bootstrap: bool = True,
                 refresh_every: int | None = None):
        """refresh_every = R: after every R-th incremental batch the caches are rebuilt by a
        full bootstrap (SPEC.md:494 drift control; default off)."""
        if not isinstance(bundle, Bundle) or bundle.model not in MODELS:
            raise E.UnsupportedModel("engine needs a bundle from paper_2603_20622_b200.models")
        if refresh_every is not None and int(refresh_every) < 1:
            raise E.ConfigError(f"refresh_every must be >= 1, got {refresh_every}")
        self.refresh_every = None if refresh_every is None else int(refresh_every)
        self._since_refresh = 0
        self.b = bundle
        self.g = graph
        self.use_graphs = bool(use_graphs)
        self._graphs: dict = {}
        self._seen: dict = {}
        self.graph_kernels: dict = {}  # batch size -> kernel nodes of the captured step (both parts)
        self._graph_nodes: dict = {}
        # RTEC_STEP_OVERLAP=0: read the apply results back after the whole step (A/B)
        self._overlap_rb = os.environ.get("RTEC_STEP_OVERLAP", "1") != "0"
        self._host = None  # pinned result buffers of step()
        self.lib = graph.lib
        self.dev = graph.dev
        n = graph.n
        self.n = n
        dims = bundle.dims
        X = torch.as_tensor(np.asarray(features), device=self.dev) if not isinstance(features, torch.Tensor) else features
        if tuple(X.shape) != (n, dims[0]):
            raise E.ShapeError(f"features shape {tuple(X.shape)} != ({n}, {dims[0]})")
        self.H = [X.to(self.dev, torch.float32).contiguous()]
        self.L = bundle.num_layers
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=self.dev)  # noqa: E731
        self.layers, self.wt = [], []
        self.S, self.ctx, self.log = [], [], []
        self.Z, self.el, self.er, self.Zlog, self.erlog = [], [], [], [], []
        heads = bundle.heads
        no = self._rows_owned()  # rows of the destination-side state (all n unless sharded)
        # tcgen05 3xTF32 (gemm_tc.cu) for every dense contraction with d_out <= 256: the update
        # GEMM, and GAT's projection Z = W h (K13; rows packed into an A image of n rows, kept
        # under a memory budget -- beyond it the projection stays on the SIMT GEMM)
        self.tc = update == "tc" and max(dims[1:]) <= 256
        if self.tc and bundle.model == GAT:
            img_bytes = (n + 127) // 128 * 128 * ((max(dims[:-1]) + 31) // 32 * 32) * 4
            self.tc = img_bytes <= self.GAT_IMG_BUDGET
        # sum aggregators on the tcgen05 path: the update epilogue of layer l writes the source
        # deltas of layer l+1 (no DeltaLog, no per-source delta pass over V_chg(l))
        self.fused = (self.FUSED_DELTA and self.tc and bundle.model in (GCN, GRAPHSAGE, GIN)
                      and all(d % 4 == 0 for d in dims[1:-1]))
        # one vertex-indexed δ buffer shared by all layers: layer l's rows are dead once its
        # aggregation has run, before the update epilogue writes layer l+1's (stream order)
        self.delta = [None] * bundle.num_layers
        if self.fused:
            dbuf = z(n * max(bundle.agg_dims))
            self.delta = [dbuf[: n * d].view(n, d) for d in bundle.agg_dims]
        for l, w in enumerate(bundle.layers):
            d_in, d_out = w.in_dim, w.out_dim
            dev32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32), device=self.dev)  # noqa: E731
            t = w.tensors
            Wnp = np.asarray(t["W"], np.float64)
            if bundle.model == COMMNET:  # W h_v + W2 a_v == [W | W2] [h_v ; a_v]
                Wnp = np.concatenate([Wnp, np.asarray(t["W2"], np.float64)], 1)
            W = dev32(Wnp)
            W2 = dev32(t["W2"]) if bundle.model in GIN_FAMILY else None
            att = dev32(np.asarray(t["a"]).reshape(heads, -1)) if bundle.model == GAT else None
            Wp = bp = None
            scalar = 0.0
            if bundle.model == PINSAGE:  # alpha relu(Q h + q)
                Wp, bp, scalar = dev32(t["Q"]), dev32(t["q"]), float(w.scalars.get("alpha", 1.0))
            elif bundle.model == MONET:  # the quadratic form only sees the symmetric part of Wq
                Wq = np.asarray(t["Wq"], np.float64)
                Wp, bp = dev32(0.5 * (Wq + Wq.T)), dev32(t["mu"])
            elif bundle.model == GGCN:
                Wp = dev32(np.concatenate([np.asarray(t["Wg_src"]), np.asarray(t["Wg_dst"])], 0))
            elif bundle.model == AGNN:
                scalar = float(w.scalars["beta"])
            d_k = bundle.update_width(l)
            tcw = [None, None, None, None]
            if self.tc:  # GAT: the operand images of the projection W [d_out, d_in]
                tcw[0], tcw[1] = self._prep_weights(W, d_in if bundle.model == GAT else d_k, d_out)
                if W2 is not None:
                    tcw[2], tcw[3] = self._prep_weights(W2, d_out, d_out)
            self.wt.append((W, W2, att, *tcw, Wp, bp))
            p = _lib.ptr
            self.layers.append(_lib.Layer(_MODEL_ID[bundle.model], d_in, d_out, heads if bundle.model == GAT else 1,
                                          float(bundle.degree_offset), 0, p(W), p(W2), p(att),
                                          p(tcw[0]), p(tcw[1]), p(tcw[2]), p(tcw[3]), p(Wp), p(bp), scalar, d_k))
            d_agg = bundle.agg_dims[l]
            # layer inputs are read for every source: full rows; the final output only per owner
            self.H.append(z(n if l + 1 < bundle.num_layers else no, d_out))
            self.S.append(z(no, d_agg))
            # DeltaLog of this layer's output (rows = V_dst slots); the final layer's is never read
            self.log.append(z(no, d_out) if l + 1 < bundle.num_layers and not self.fused else None)
            if bundle.model == GAT:
                self.ctx.append(z(no, heads))
                self.Z.append(z(n, d_out))
                self.el.append(z(n, heads))
                self.er.append(z(n, heads))
                self.Zlog.append(z(n, d_out))
                self.erlog.append(z(n, heads))
            elif bundle.projected:  # payload / gate projections of every vertex + their batch log
                pw = bundle.proj_width(l)
                self.ctx.append(None)
                self.Z.append(z(n, pw))
                self.Zlog.append(z(n, pw))
                for lst in (self.el, self.er, self.erlog):
                    lst.append(None)
            else:
                self.ctx.append(None)
                for lst in (self.Z, self.el, self.er, self.Zlog, self.erlog):
                    lst.append(None)
        self.max_dim = max(max(dims), 1)
        pad = lambda d: (d + 31) // 32 * 32  # noqa: E731
        if self.tc and bundle.model == GAT:  # projection A image over every row (bootstrap, replicas)
            self.gemm_in = z((n + 127) // 128 * 128 * pad(max(dims[:-1])))
            self.gemm_mid = None
        elif self.tc:  # SW128 tile image: ceil(rows/128)*128 rows x ceil(d/32)*32 columns
            rows = (no + 127) // 128 * 128
            self.gemm_in = z(rows * pad(max(bundle.update_width(l) for l in range(self.L))))
            self.gemm_mid = z(rows * pad(max(dims[1:]))) if bundle.model in GIN_FAMILY else None
        else:
            self.gemm_in = z(no, max(bundle.update_width(l) for l in range(self.L))) if bundle.model != GAT else None
            self.gemm_mid = z(no, max(dims[1:])) if bundle.model in GIN_FAMILY else None
        self.fr = [_Frontier(n, self.dev) for _ in range(self.L)]
        self._ensure_ws(max_batch or graph.batch.cap)
        if bootstrap:  # (formats.load_checkpoint restores the state instead)
            self.bootstrap()

    # ---------------------------------------------------------------- plumbing
    def _rows_owned(self) -> int:
        """Rows of the destination-side state (S, ctx, final H, DeltaLog, GEMM input)."""
        return self.n

    def _prep_weights(self, W, d_in, d_out):
        nkb, npad = (d_in + 31) // 32, (d_out + 15) // 16 * 16
        hi = torch.zeros(nkb * npad * 32, dtype=torch.float32, device=self.dev)
        lo = torch.zeros_like(hi)
        _lib.check(self.lib.rtec_gemm_prepare_weights(_lib.ptr(W), d_in, d_out, _lib.ptr(hi), _lib.ptr(lo),
                                                      _lib.stream_handle()), "prepare_weights")
        return hi, lo

    def _ensure_ws(self, B):
        need = int(self.lib.rtec_workspace_bytes(self.n, max(int(B), 1), max(self.g.out.slots, self.g.inn.slots),
                                                 self.max_dim))
        if self.g.ws.numel() < need:
            self.g.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)

    def _state(self, l, incremental: bool = False):
        p = _lib.ptr
        st = _lib.State(p(self.H[l]), p(self.H[l + 1]), p(self.S[l]), p(self.ctx[l]), p(self.log[l]),
                        p(self.log[l - 1]) if l > 0 else None, p(self.Z[l]), p(self.el[l]), p(self.er[l]),
                        p(self.Zlog[l]), p(self.erlog[l]), p(self.gemm_in), p(self.gemm_mid))
        if incremental and self.fused:
            st.delta = p(self.delta[l])
            st.delta_next = p(self.delta[l + 1]) if l + 1 < self.L else None
            st.delta_ready = 1 if l > 0 else 0
        return st

    # ---------------------------------------------------------------- SPEC bootstrap / run_full
    def bootstrap(self, sync: bool = True):
        """Full forward populating every layer's state (models.py:461-477);
        also SPEC run_full on the current graph."""
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        g = self.g.c()
        st = _lib.stream_handle()
        for l in range(self.L):
            s = self._state(l)
            _lib.check(self.lib.rtec_layer_full(C.byref(g), C.byref(self.layers[l]), C.byref(s), None, None, self.n,
                                                _lib.ptr(err), _lib.ptr(self.g.ws), self.g.ws.numel(), st), "bootstrap")
        if sync:
            _lib.raise_err(err.item(), "bootstrap")

    def _project(self, l, H, rows, n_rows, Z, el=None, er=None, Zlog=None, erlog=None, err=None, stream=None):
        """Per-vertex projections of layer l for `rows` (all when None) from H: GAT Z / el / er
        (rtec_gat_project), PinSAGE / MoNet payloads and G-GCN gates (rtec_project)."""
        p = _lib.ptr
        st = stream if stream is not None else _lib.stream_handle()
        if self.b.model == GAT:
            _lib.check(self.lib.rtec_gat_project(C.byref(self.layers[l]), p(H), p(rows), p(n_rows), self.n, p(Z),
                                                 p(el), p(er), p(Zlog), p(erlog), p(err), self._proj_img(), st),
                       "gat_project")
        elif self.b.projected:
            _lib.check(self.lib.rtec_project(C.byref(self.layers[l]), p(H), p(rows), p(n_rows), self.n, p(Z),
                                             p(Zlog), p(err), st), "project")

    def _proj_img(self):
        """A-image scratch of the tcgen05 GAT projection (None: SIMT)."""
        return _lib.ptr(self.gemm_in) if (self.tc and self.b.model == GAT) else None

    def refresh_projection(self, l: int) -> None:
        """Projections of every vertex of layer l from H^l (after a restore)."""
        if self.b.projected:
            self._project(l, self.H[l], None, None, self.Z[l], self.el[l], self.er[l])

    def save(self, directory: str) -> None:
        """Checkpoint between batches (formats.save_checkpoint)."""
        from .formats import save_checkpoint

        save_checkpoint(self, directory)

    @staticmethod
    def load(directory: str, **kw) -> "RTECEngine":
        """Resume from a checkpoint without a bootstrap (formats.load_checkpoint)."""
        from .formats import load_checkpoint

        return load_checkpoint(directory, **kw)

    def run_full(self, batch=None) -> RunResult | None:
        """SPEC run_full: without a batch, recompute every layer on the
        current graph; with one, apply it and recompute everything (the RTEC-Full baseline)."""
        if batch is None:
            self.bootstrap()
            return None
        return self.step(*updates_to_arrays(list(batch)), mode="full")

    # ---------------------------------------------------------------- incremental step
    def _graph_key(self, B: int):
        """Everything a captured step bakes in: the batch size and the graph's buffer layout --
        DynamicGraph.layout_version moves whenever a run array, degree array, the batch buffers
        or the workspace is rebound (compaction, a larger batch, workspace growth), so a graph
        is never replayed against moved or freed buffers (the engine's own tensors are fixed)."""
        gr = self.g
        return (B, id(gr), gr.layout_version, gr.ws.data_ptr())

    def enqueue_step(self, B: int) -> None:
        """Enqueue the whole incremental pipeline for the staged batch (no sync): part 1 the
        apply chain (statuses, DegreeDelta rows final), part 2 frontiers, layers and commit.

        With `use_graphs`, each part (~100-200 launches together) is captured into a CUDA
        graph on the second batch of a given size and replayed afterwards; any
        reallocation (workspace growth, compaction, larger batch buffers) changes
        the key and triggers a fresh capture.  step() reads the apply results back
        between the two parts, under part 2's compute."""
        self._enqueue_part(B, 1)
        self._enqueue_part(B, 2)

    def _enqueue_part(self, B: int, part: int) -> None:
        self._ensure_ws(self.g.batch.cap)
        run = (lambda: self.g.apply_staged(B)) if part == 1 else (lambda: self._enqueue_layers(B))
        if not self.use_graphs:
            run()
            return
        key = self._graph_key(B) + (part,)
        cg = self._graphs.get(key)
        if cg is None:
            if self._seen.get(key, 0) < 1:  # first batch of this shape runs eagerly (lazy init, warm-up)
                self._seen[key] = self._seen.get(key, 0) + 1
                run()
                return
            prof = _lib.prof_enabled()
            self.lib.rtec_prof_enable(0)
            cg = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(cg):
                run()
            cg.instantiate()
            self.lib.rtec_prof_enable(1 if prof else 0)
            self._graph_nodes[key] = int(self.lib.rtec_graph_kernel_nodes(cg.raw_cuda_graph()))
            self.graph_kernels[B] = sum(v for k, v in self._graph_nodes.items() if k[0] == B)
            if len(self._graphs) >= 8:
                self._graphs.pop(next(iter(self._graphs)))
            self._graphs[key] = cg
        cg.replay()

    def _enqueue_eager(self, B: int, mode: str = "inc") -> None:
        """mode 'inc': Alg. 1 / Alg. 3 (run_incremental); 'uer': the same affected rows
        recomputed over their full in-neighbourhoods (SPEC.md:455 run_uer)."""
        self.g.apply_staged(B)
        self._enqueue_layers(B, mode)

    def _enqueue_layers(self, B: int, mode: str = "inc") -> None:
        """Frontiers, layers and the batch commit for the applied batch (after apply_staged)."""
        gr = self.g
        g, b = gr._gc, gr._bc
        st = _lib.stream_handle()
        ws, wsb = _lib.ptr(gr.ws), gr.ws.numel()
        errp = _lib.ptr(gr.batch.err)
        sdd = 1 if self.b.src_degree_dependent else 0
        self._fc = [f.c() for f in self.fr]
        self._sc = [self._state(l, incremental=True) for l in range(self.L)]
        # The frontier of layer l+1 needs only layer l's frontier, not its embeddings: layers
        # 1..L-1's frontiers run on a side stream (own workspace) under layer 0's compute and
        # each layer waits for its frontier (a fork / join the CUDA graph keeps).
        overlap = mode != "frontier" and self.L > 1
        main = torch.cuda.current_stream()
        _lib.check(self.lib.rtec_frontier_layer(C.byref(g), C.byref(b), 0, sdd, None, C.byref(self._fc[0]), ws, wsb,
                                                st), "frontier")
        if overlap:  # fork after layer 0's frontier
            fws = self._frontier_ws()
            side, evs = self._side()
            evs[0].record(main)
            side.wait_event(evs[0])
            with torch.cuda.stream(side):
                for l in range(1, self.L):
                    _lib.check(self.lib.rtec_frontier_layer(C.byref(g), C.byref(b), l, sdd, C.byref(self._fc[l - 1]),
                                                            C.byref(self._fc[l]), _lib.ptr(fws), fws.numel(),
                                                            side.cuda_stream), "frontier")
                    evs[l].record(side)
        for l in range(self.L):
            prev = C.byref(self._fc[l - 1]) if l > 0 else None
            if l > 0 and not overlap:
                _lib.check(self.lib.rtec_frontier_layer(C.byref(g), C.byref(b), l, sdd, prev, C.byref(self._fc[l]), ws,
                                                        wsb, st), "frontier")
            elif l > 0:
                main.wait_event(self._side()[1][l])
            if mode == "frontier":
                continue
            if self.b.projected and l > 0:  # projections of the rows V_chg(l-1) rewrote (+ their log)
                pf = self.fr[l - 1]
                self._project(l, self.H[l], pf.dst_list, pf.n_dst, self.Z[l], self.el[l], self.er[l], self.Zlog[l],
                              self.erlog[l], gr.batch.err, st)
            if mode == "uer":
                f = self.fr[l]
                s_full = self._state(l)
                _lib.check(self.lib.rtec_layer_full(C.byref(g), C.byref(self.layers[l]), C.byref(s_full),
                                                    _lib.ptr(f.dst_list), _lib.ptr(f.n_dst), self.n, errp, ws, wsb,
                                                    st), "layer (uer)")
            else:
                _lib.check(self.lib.rtec_layer_incremental(C.byref(g), C.byref(b), C.byref(self.layers[l]),
                                                           C.byref(self._sc[l]), prev, C.byref(self._fc[l]), errp, ws,
                                                           wsb, st), "layer")
        _lib.check(self.lib.rtec_batch_commit(C.byref(g), C.byref(b), st), "commit")

    def _side(self):
        if getattr(self, "_side_stream", None) is None:
            self._side_stream = torch.cuda.Stream(device=self.dev)
            self._side_events = [torch.cuda.Event() for _ in range(self.L)]
        return self._side_stream, self._side_events

    def _frontier_ws(self) -> torch.Tensor:
        need = int(self.n) * 24 + (1 << 20)  # list + offsets + word offsets + scan partials
        if getattr(self, "_fws", None) is None or self._fws.numel() < need:
            self._fws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        return self._fws

    def _host_buffers(self):
        cap = self.g.batch.cap
        hb = self._host
        if hb is None or hb["cap"] < cap:
            pin = lambda t, k: torch.empty(k, dtype=t, pin_memory=True)  # noqa: E731
            hb = self._host = {"cap": cap, "err": pin(torch.int64, 1), "nd": pin(torch.int64, 1),
                               "status": pin(torch.uint8, cap),
                               "d": torch.empty((2 * cap, 5), dtype=torch.int32, pin_memory=True),
                               "ctr": pin(torch.int64, 8 * self.L)}
        return hb

    def _readback_apply(self, hb, B: int) -> None:
        """Queue the apply results (DegreeDelta count, statuses, DegreeDelta rows) into the
        pinned buffers on the current stream."""
        b = self.g.batch
        hb["nd"].copy_(b.n_delta, non_blocking=True)
        if B:
            hb["status"][:B].copy_(b.status[:B], non_blocking=True)
            # DegreeDelta rows (at most 2B) interleaved into [rows, 5] on the device: one copy,
            # and the host result is a slice instead of a stack of five columns
            hb["d"][: 2 * B].copy_(torch.stack([t[: 2 * B] for t in b.d], dim=1), non_blocking=True)

    def _readback_tail(self, hb) -> None:
        """Queue the error word and the frontier counters (after the layers)."""
        hb["err"].copy_(self.g.batch.err, non_blocking=True)
        for l, f in enumerate(self.fr):
            hb["ctr"][8 * l: 8 * l + 8].copy_(f.counters, non_blocking=True)

    def _readback(self, B: int):
        """Queue the batch's results into pinned host buffers (one sync for all of them)."""
        hb = self._host_buffers()
        self._readback_apply(hb, B)
        self._readback_tail(hb)
        torch.cuda.current_stream().synchronize()
        return hb

    def _step_overlapped(self, B: int):
        """The incremental step with its apply results read back under the layer compute:
        part 1 (apply chain), then on a side stream the D2H of statuses and DegreeDelta
        rows, then part 2 (frontiers, layers, commit) on the main stream; the host turns
        the apply results into arrays while part 2 runs, and waits for the main stream
        only for the error word and counters."""
        hb = self._host_buffers()
        main = torch.cuda.current_stream()
        self._enqueue_part(B, 1)
        if getattr(self, "_rb_stream", None) is None:
            self._rb_stream = torch.cuda.Stream(device=self.dev)
            self._rb_events = (torch.cuda.Event(), torch.cuda.Event())
        side, (e_apply, e_rb) = self._rb_stream, self._rb_events
        e_apply.record(main)
        side.wait_event(e_apply)
        with torch.cuda.stream(side):
            self._readback_apply(hb, B)
        e_rb.record(side)
        self._enqueue_part(B, 2)
        self._readback_tail(hb)
        main.wait_event(e_rb)  # the side copies finish before the main stream moves on
        e_rb.synchronize()
        status = hb["status"][:B].numpy().copy()
        k = int(hb["nd"][0])
        deltas = hb["d"][:k].numpy().copy() if k else np.zeros((0, 5), np.int32)
        main.synchronize()
        return hb, status, deltas

    def _metrics_from(self, ctr, mode: str = "inc") -> Metrics:
        m = Metrics(mode=mode)
        c = ctr.numpy().reshape(self.L, 8)
        m_edges = self.g.num_edges if mode == "full" else 0
        for l in range(self.L):
            m.e_curr.append(int(c[l, 0]))
            m.v_dst.append(int(c[l, 1]))
            m.n_src.append(int(c[l, 2]))
            m.in_edges_vdst.append(int(c[l, 5]))
            # access counters: one edge access per processed (edge, layer),
            # one vertex access per recomputed destination
            if mode == "inc":
                m.edge_accesses.append(int(c[l, 0]))
                m.vertex_accesses.append(int(c[l, 1]))
            elif mode == "odec":  # deferred: no layer work at batch time
                m.edge_accesses.append(0)
                m.vertex_accesses.append(0)
            elif mode == "ns":  # sampled edges / rows of hop l
                m.edge_accesses.append(int(self._ns["adj"][l]["top"].item()))
                m.vertex_accesses.append(int(self._ns["cnt"][l + 1].item()) if l + 1 < self.L else int(c[l, 1]))
            elif mode == "uer":
                m.edge_accesses.append(int(c[l, 5]))
                m.vertex_accesses.append(int(c[l, 1]))
            else:
                m.edge_accesses.append(int(m_edges))
                m.vertex_accesses.append(int(self.n))
        m.as_edges = sum(m.e_curr)
        m.as_vertices = sum(m.v_dst)
        return m

    # ---------------------------------------------------------------- NS baseline
    def _ns_buffers(self, fanout: int):
        nb = getattr(self, "_ns", None)
        if nb is not None and nb["fanout"] >= fanout:
            return nb
        n, dev, L = self.n, self.dev, self.L
        words = (n + 31) // 32
        zi = lambda k, dt=torch.int32: torch.zeros(max(k, 1), dtype=dt, device=dev)  # noqa: E731
        zf = lambda *sh: torch.zeros(*sh, dtype=torch.float32, device=dev)  # noqa: E731
        nb = {"fanout": fanout,
              "bm": [zi(words) for _ in range(L)], "T": [zi(n) for _ in range(L)],
              "cnt": [zi(1, torch.int64) for _ in range(L)],
              "adj": [{"beg": zi(n, torch.int64), "len": zi(n), "nbr": zi(n * fanout), "top": zi(1, torch.int64)}
                      for _ in range(L)],
              "H": [None] + [zf(n, d) for d in self.b.dims[1:]],
              "S": zf(n, max(self.b.agg_dims)),
              "Z": (zf(n, max(self.b.dims[1:])) if self.b.model == GAT else
                    zf(n, max(self.b.proj_width(l) for l in range(L))) if self.b.projected else None),
              "el": zf(n, self.b.heads) if self.b.model == GAT else None,
              "er": zf(n, self.b.heads) if self.b.model == GAT else None,
              "ctx": zf(n, self.b.heads) if self.b.model == GAT else None}
        self._ns = nb
        return nb

    def _ns_enqueue(self, fanout: int, seed: int) -> None:
        """SPEC run_ns (§III-B): the final-layer affected vertices of the
        batch (V_dst(L-1)) recomputed over L-hop in-neighbourhoods sampled without
        replacement, at most `fanout` per vertex per hop, seeded; approximate by design.  The
        result overwrites those rows of the final embeddings only (the exact caches are not
        maintained: run NS on its own engine)."""
        nb = self._ns_buffers(fanout)
        lib, p, st = self.lib, _lib.ptr, _lib.stream_handle()
        gr = self.g
        ws, wsb = p(gr.ws), gr.ws.numel()
        n, L = self.n, self.L
        rows, cnt = self.fr[L - 1].dst_list, self.fr[L - 1].n_dst  # T_L
        T, C_ = [None] * (L + 1), [None] * (L + 1)
        T[L], C_[L] = rows, cnt
        adjs = []
        for l in range(L - 1, -1, -1):  # sample downwards: T_l = T_{l+1} ∪ sampled in-neighbours
            a = nb["adj"][l]
            smp = _lib.Adj(a["nbr"].numel(), p(a["beg"]), p(a["len"]), None, p(a["nbr"]), None, p(a["top"]))
            inn = gr.inn.c()
            _lib.check(lib.rtec_ns_sample(C.byref(inn), p(T[l + 1]), p(C_[l + 1]), n, int(fanout),
                                          C.c_uint64(int(seed) & ((1 << 64) - 1)), l, C.byref(smp), p(nb["bm"][l]),
                                          n, ws, wsb, st), "ns_sample")
            _lib.check(lib.rtec_bitmap_to_list(p(nb["bm"][l]), n, p(nb["T"][l]), p(nb["cnt"][l]), ws, wsb, st),
                       "ns_rows")
            T[l], C_[l] = nb["T"][l], nb["cnt"][l]
            adjs.append(smp)
        adjs.reverse()  # adjs[l] = sampled in-neighbours of T_{l+1}
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        H = [self.H[0]] + nb["H"][1:]
        for l in range(L):
            g = gr.c()
            g.inn = adjs[l]
            s = self._state(l)
            s.H_in, s.H_out, s.S = p(H[l]), p(H[l + 1]), p(nb["S"])
            s.log_out = s.log_in = None
            if self.b.projected:  # projections of the sampled rows T_l
                s.Z, s.el, s.er, s.ctx = p(nb["Z"]), p(nb["el"]), p(nb["er"]), p(nb["ctx"])
                s.Z_log = s.er_log = None
                self._project(l, H[l], T[l], C_[l], nb["Z"], nb["el"], nb["er"], err=err, stream=st)
            _lib.check(lib.rtec_layer_full(C.byref(g), C.byref(self.layers[l]), C.byref(s), p(T[l + 1]),
                                           p(C_[l + 1]), n, p(err), ws, wsb, st), "ns_layer")
        k = int(cnt.item())
        if k:
            idx = rows[:k].to(torch.int64)
            self.H[L][idx] = H[L][idx]

    def run_ns(self, batch, fanout: int = 10, seed: int = 0) -> RunResult:
        """SPEC run_ns on a coalesced EdgeUpdate list."""
        return self.step(*updates_to_arrays(list(batch)), mode="ns", fanout=fanout, seed=seed)

    # ---------------------------------------------------------------- ODEC (query-driven)
    def _odec_state(self):
        if getattr(self, "_stale", None) is None:
            words = (self.n + 31) // 32
            z = lambda: torch.zeros(max(words, 1), dtype=torch.int32, device=self.dev)  # noqa: E731
            self._stale = [z() for _ in range(self.L)]  # rows of H^{l+1} / S^l whose cache is out of date
            self._need = [z() for _ in range(self.L)]
            self._rows = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.dev)
            self._nrows = torch.zeros(1, dtype=torch.int64, device=self.dev)
        return self._stale

    def odec_flush(self) -> None:
        """Recompute every deferred row (then any engine mode may follow)."""
        if getattr(self, "_stale", None) is None:
            return
        lib, p, st = self.lib, _lib.ptr, _lib.stream_handle()
        gr = self.g
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        prev = None
        for l in range(self.L):
            if self.b.projected and l > 0 and prev is not None:
                self._project(l, self.H[l], prev[0], prev[1], self.Z[l], self.el[l], self.er[l])
            rows = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.dev)
            nrows = torch.zeros(1, dtype=torch.int64, device=self.dev)
            _lib.check(lib.rtec_bitmap_to_list(p(self._stale[l]), self.n, p(rows), p(nrows), p(gr.ws), gr.ws.numel(),
                                               st), "odec")
            _lib.check(lib.rtec_layer_full(C.byref(gr.c()), C.byref(self.layers[l]), C.byref(self._state(l)), p(rows),
                                           p(nrows), self.n, p(err), p(gr.ws), gr.ws.numel(), st), "odec")
            self._stale[l].zero_()
            prev = (rows, nrows)
        _lib.raise_err(err.item(), "odec_flush")

    def stale_rows(self, l: int) -> int:
        """ODEC: vertices whose layer-l output is deferred (cache out of date)."""
        st = self._odec_state()[l]
        return int(torch.bitwise_count(st.view(torch.int32)).sum().item()) if hasattr(torch, "bitwise_count") \
            else int(sum(bin(int(w) & 0xFFFFFFFF).count("1") for w in st.cpu().tolist()))

    def _mark(self, bm: torch.Tensor, ids: torch.Tensor) -> None:
        """bm |= bits of the (device) ids."""
        u = torch.unique(ids.to(torch.int64))
        w = torch.zeros(bm.numel(), dtype=torch.int64, device=self.dev)
        w.index_add_(0, u >> 5, torch.ones_like(u) << (u & 31))  # distinct bits: add == or
        bm |= w.to(torch.int32)

    def odec_query(self, ids) -> np.ndarray:
        """SPEC run_odec (§V-D): fresh final-layer rows of `ids`.
        Batches applied with mode 'odec' only mark the affected rows of every layer as
        deferred; a query recomputes, bottom-up, the deferred rows inside the queries' L-hop
        in-subgraph over their full post-batch in-neighbourhoods, clears their staleness and
        returns H^L[ids] -- equal to a full recomputation on the current graph."""
        stale = self._odec_state()
        ids_np = np.asarray(ids, np.int64).reshape(-1)
        if ids_np.size and (ids_np.min() < 0 or ids_np.max() >= self.n):
            raise E.InvalidVertex("query vertex outside the vertex range")
        if ids_np.size == 0:
            return np.zeros((0, self.b.dims[-1]), np.float32)
        lib, p, st = self.lib, _lib.ptr, _lib.stream_handle()
        gr = self.g
        inn = gr.inn.c()
        L, n = self.L, self.n
        q = torch.as_tensor(ids_np.astype(np.int32), device=self.dev)
        # need[l]: rows whose layer-l output the queries depend on; need[l-1] = need[l] ∪ in-nbrs
        for b in self._need:
            b.zero_()
        self._mark(self._need[L - 1], q)
        for l in range(L - 1, 0, -1):
            _lib.check(lib.rtec_bitmap_to_list(p(self._need[l]), n, p(self._rows), p(self._nrows), p(gr.ws),
                                               gr.ws.numel(), st), "odec")
            _lib.check(lib.rtec_in_expand(C.byref(inn), p(self._rows), p(self._nrows), n, p(self._need[l - 1]), st),
                       "odec")
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        prev_rows = None
        for l in range(L):  # bottom-up over the deferred rows the queries need
            if self.b.projected and l > 0 and prev_rows is not None:  # fresh H^l rows: fresh projections
                self._project(l, self.H[l], prev_rows[0], prev_rows[1], self.Z[l], self.el[l], self.er[l])
            todo = stale[l] & self._need[l]
            rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
            nrows = torch.zeros(1, dtype=torch.int64, device=self.dev)
            _lib.check(lib.rtec_bitmap_to_list(p(todo), n, p(rows), p(nrows), p(gr.ws), gr.ws.numel(), st), "odec")
            s_full = self._state(l)
            _lib.check(lib.rtec_layer_full(C.byref(gr.c()), C.byref(self.layers[l]), C.byref(s_full), p(rows),
                                           p(nrows), n, p(err), p(gr.ws), gr.ws.numel(), st), "odec")
            stale[l] &= ~todo
            prev_rows = (rows, nrows)
        _lib.raise_err(err.item(), "odec_query")
        return self.H[L][q.to(torch.int64)].cpu().numpy()

    def run_uer(self, batch) -> RunResult:
        """SPEC run_uer: affected rows over their full in-neighbourhoods."""
        return self.step(*updates_to_arrays(list(batch)), mode="uer")

    def step(self, op, src, dst, ts, mode: str = "inc", fanout: int = 10, seed: int = 0) -> RunResult:
        """One batch on array inputs: mode 'inc' = run_incremental, 'uer' =
        run_uer, 'full' = apply + run_full.  One host
        synchronisation at the end reads the per-update status, DegreeDelta rows and
        counters from pinned buffers."""
        if mode not in ("inc", "uer", "full", "ns", "odec"):
            raise E.ConfigError(f"unknown engine mode {mode!r} (inc, uer, full, ns, odec)")
        t0 = time.perf_counter()
        if mode != "odec" and getattr(self, "_stale", None) is not None and any(int(b.any()) for b in self._stale):
            raise E.StaleState("deferred (ODEC) rows pending: call odec_flush() before another mode")
        B = self.g.stage(op, src, dst, ts)
        for attempt in range(4):
            early = None
            if mode == "inc" and self._overlap_rb:
                hb, *early = self._step_overlapped(B)
            elif mode == "inc":
                self.enqueue_step(B)
            else:
                self._ensure_ws(self.g.batch.cap)
                # 'full' / 'ns': apply + the frontier (access counters, affected final rows)
                self._enqueue_eager(B, mode="uer" if mode == "uer" else "frontier")
                if mode == "full":
                    self.bootstrap(sync=False)
                elif mode == "ns":
                    self._ns_enqueue(fanout, seed)
                elif mode == "odec":  # defer: the affected rows of every layer become stale
                    stale = self._odec_state()
                    for l in range(self.L):
                        stale[l] |= self.fr[l].bm_dst
            if early is None:
                hb = self._readback(B)
            word = int(hb["err"][0]) & _lib.ERR_OK
            d = _lib.decode_err(word)
            if d is not None and d[0] == _lib.ARENA_FULL:
                # nothing was mutated (validation-before-mutation); make room and replay
                self.g.compact(min_reserve=(16 * B + 4096) * 4 ** attempt)
                self.g._ensure_ws(self.g.batch.cap, grow=2.0 ** (attempt + 1))
                self._ensure_ws(self.g.batch.cap)
                continue
            _lib.raise_err(word, "run_incremental", self.g._ERR_MSG)
            break
        else:
            raise E.NativeError("run_incremental: arena still full after compaction")
        if early is not None:
            status, deltas = early
        else:
            status = hb["status"][:B].numpy().copy()
            k = int(hb["nd"][0])
            # DegreeDelta rows (vertex, old_in, new_in, old_out, new_out) as int32 [k, 5]
            deltas = hb["d"][:k].numpy().copy() if k else np.zeros((0, 5), np.int32)
        m = self._metrics_from(hb["ctr"], mode)
        changed = self._changed_final(mode, m)
        if mode in ("inc", "uer") and self.refresh_every:
            self._since_refresh += 1
            if self._since_refresh >= self.refresh_every:  # SPEC.md:494 drift control
                self.bootstrap()
                self._since_refresh = 0
                m.refreshed = True
        elif mode == "full":
            self._since_refresh = 0
        m.wall_time = time.perf_counter() - t0
        return RunResult(status, deltas, changed, m)

    def _changed_final(self, mode: str, m: Metrics):
        """Device snapshot of the ids whose final-layer rows this step recomputed."""
        if mode == "odec":
            return np.zeros(0, np.int64)
        if mode == "full":
            return torch.arange(self.n, dtype=torch.int64, device=self.dev)
        k = m.v_dst[-1] if m.v_dst else 0
        return self.fr[-1].dst_list[:k].clone()

    def run_incremental(self, batch) -> RunResult:
        """SPEC run_incremental on a coalesced EdgeUpdate list."""
        return self.step(*updates_to_arrays(list(batch)))

    # ---------------------------------------------------------------- reads
    def metrics(self) -> Metrics:
        m = Metrics()
        for f in self.fr:
            c = f.counters.cpu().numpy()
            m.e_curr.append(int(c[0]))
            m.v_dst.append(int(c[1]))
            m.n_src.append(int(c[2]))
            m.in_edges_vdst.append(int(c[5]))
        return m

    def degree_breakdown(self, shares=(0.2, 0.3, 0.5)) -> dict:
        """Table V / SPEC.md:564 degree-percentile breakdown of the LAST batch's edge accesses:
        vertices ranked by in-degree (descending, ties by id) into top 20 % / mid 30 % /
        bottom 50 %; each edge access is charged to its destination's class.  FN = every
        in-edge at every layer, UER = in-runs of V_dst(l), Inc = E_curr(l) (G_post out-edges of
        S(l), plus applied inserts from other sources and deletes).  Device torch ops over
        the frontier lists and adjacency; Σ over classes of `inc` equals Σ_l |E_curr(l)|."""
        n, L, dev = self.n, self.L, self.dev
        gr = self.g
        indeg = gr.in_deg[:n].to(torch.int64)
        order = torch.argsort(-indeg, stable=True)
        cls = torch.empty(n, dtype=torch.int64, device=dev)
        cuts = np.ceil(np.cumsum(shares) * n).astype(np.int64).tolist()
        lo = 0
        for c, hi in enumerate(cuts):
            cls[order[lo:min(hi, n)]] = c
            lo = min(hi, n)
        nc = len(shares)
        cnt = lambda idx, w=None: torch.bincount(cls[idx], weights=w, minlength=nc)  # noqa: E731
        fn = L * torch.bincount(cls, weights=indeg.to(torch.float64), minlength=nc)
        uer = torch.zeros(nc, dtype=torch.float64, device=dev)
        inc = torch.zeros(nc, dtype=torch.float64, device=dev)
        b = gr.batch
        na = int(b.n_applied.item())
        a_src, a_dst = b.a_src[:na].to(torch.int64), b.a_dst[:na].to(torch.int64)
        ins = b.a_op[:na] == _lib.OP_INSERT
        for l in range(L):
            f = self.fr[l]
            ns, nd = int(f.n_src.item()), int(f.n_dst.item())
            S = f.src_list[:ns].to(torch.int64)
            V = f.dst_list[:nd].to(torch.int64)
            uer += cnt(V, indeg[V].to(torch.float64))
            lens = gr.out.len[S].to(torch.int64)
            tot = int(lens.sum().item()) if ns else 0
            if tot:
                start = torch.repeat_interleave(gr.out.beg[S] - (torch.cumsum(lens, 0) - lens), lens)
                w = gr.out.nbr[start + torch.arange(tot, device=dev)].to(torch.int64)
                inc += cnt(w).to(torch.float64)
            in_s = torch.zeros(n, dtype=torch.bool, device=dev)
            in_s[S] = True
            inc += cnt(a_dst[ins & ~in_s[a_src]]).to(torch.float64)
            inc += cnt(a_dst[~ins]).to(torch.float64)
        names = [f"{'top' if i == 0 else 'bottom' if i == nc - 1 else 'mid'}{round(100 * x)}" for i, x in enumerate(shares)]
        fn_, uer_, inc_ = (x.cpu().numpy() for x in (fn, uer, inc))
        return {"classes": names, "fn_edges": fn_.astype(np.int64).tolist(), "uer_edges": uer_.astype(np.int64).tolist(),
                "inc_edges": inc_.astype(np.int64).tolist(),
                "fn_over_inc": [float(a / c) if c else None for a, c in zip(fn_, inc_)]}

    def frontier(self, l: int):
        """(V_dst(l), S(l)) ascending id arrays of the last batch."""
        f = self.fr[l]
        nd, ns = int(f.n_dst.item()), int(f.n_src.item())
        return f.dst_list[:nd].cpu().numpy().astype(np.int64), f.src_list[:ns].cpu().numpy().astype(np.int64)

    def embeddings(self, l: int) -> np.ndarray:
        """H^l (l = 0 features, l = L final layer) as float32 numpy."""
        return self.H[l].cpu().numpy()

    def aggregates(self, l: int) -> np.ndarray:
        """Composed aggregate a^l = ms_cbn(ctx, S^l) for every vertex (reference layout)."""
        S = self.S[l]
        indeg = self.g.in_deg[: self.n].to(torch.float32)
        if self.b.model == GAT:
            h = self.b.heads
            ctx = self.ctx[l]
            safe = torch.where(ctx > 0, ctx, torch.ones_like(ctx))
            A = (S.view(self.n, h, -1) / safe[:, :, None]).reshape(self.n, -1)
        elif self.b.model == "gcn":
            A = S / torch.sqrt(indeg + self.b.degree_offset)[:, None]
        elif self.b.model in (GRAPHSAGE, PINSAGE):
            A = S / torch.clamp(indeg, min=1.0)[:, None]
        else:
            A = S
        A = torch.where((indeg > 0)[:, None], A, torch.zeros_like(A))
        return A.cpu().numpy()

    def contexts(self, l: int) -> np.ndarray:
        indeg = self.g.in_deg[: self.n].cpu().numpy().astype(np.float64)
        if self.b.model == GAT:
            c = self.ctx[l].cpu().numpy().astype(np.float64)
            return c[:, 0] if self.b.heads == 1 else c
        if self.b.ctx_kind == "count":
            return indeg
        return np.ones(self.n)

    def query(self, ids) -> np.ndarray:
        """Refreshed final-layer rows for `ids` (SPEC materialize_h SPEC.md:379)."""
        ids_t = torch.as_tensor(np.asarray(ids, np.int64), device=self.dev)
        if ids_t.numel() and (int(ids_t.min()) < 0 or int(ids_t.max()) >= self.n):
            raise E.InvalidVertex("query vertex outside the vertex range")
        ids_t = ids_t.to(torch.int32)
        d = self.b.dims[-1]
        out = torch.empty(max(ids_t.numel(), 1), d, dtype=torch.float32, device=self.dev)
        err = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
        _lib.check(self.lib.rtec_query(_lib.ptr(self.H[-1]), d, _lib.ptr(ids_t), ids_t.numel(), _lib.ptr(out), self.n,
                                       _lib.ptr(err), _lib.stream_handle()), "query")
        _lib.raise_err(err.item(), "query")
        return out[: ids_t.numel()].cpu().numpy()

    materialize_h = query


# ---------------------------------------------------------------- full-recompute API (models.py:461-492)
def _as_bundle(bundle) -> Bundle:
    if isinstance(bundle, Bundle):
        return bundle
    from .models import from_reference

    return from_reference(bundle)


def layer_embeddings(bundle, layer: int, graph: DynamicGraph, H_prev):
    """models.py:461-477 on the GPU: one full layer pass over `graph` from `H_prev`,
    returning (H_next f32[n, out], aggregates f32[n, agg], contexts f64[n]) -- the
    aggregates composed with the context (ms_cbn) exactly as the reference stores them.
    `bundle` may be ours or a reference OperatorBundle (adopted by value)."""
    b = _as_bundle(bundle)
    n = graph.num_vertices
    if not 0 <= int(layer) < b.num_layers:
        raise E.ConfigError(f"layer {layer} outside [0, {b.num_layers})")
    w = b.layers[layer]
    shape = tuple(H_prev.shape)
    if shape != (n, w.in_dim):
        raise E.ConfigError(f"layer {layer}: embeddings shape {shape} unexpected")
    from dataclasses import replace

    sub = replace(b, layers=(w,), agg_dims=(b.agg_dims[layer],))
    eng = RTECEngine(sub, graph, H_prev, use_graphs=False)
    return eng.embeddings(1), eng.aggregates(0), eng.contexts(0)


def forward_layer_reference(bundle, graph: DynamicGraph, H_prev, layer: int) -> np.ndarray:
    """models.py:480-484: H_next of one full layer."""
    return layer_embeddings(bundle, layer, graph, H_prev)[0]


def reference_embeddings(bundle, graph: DynamicGraph, features) -> np.ndarray:
    """models.py:487-492: final-layer embeddings from scratch (every layer recomputed on
    the GPU by the same full-layer kernels the engine bootstraps with)."""
    b = _as_bundle(bundle)
    eng = RTECEngine(b, graph, features, use_graphs=False)
    return eng.embeddings(b.num_layers)
