#!/usr/bin/env python
"""bench.py -- edge updates/s and p50 batch latency of the B200 incremental RTEC engine.

Default workload ("c2-gcn"): the configs[1] graph (ogbn-products shape:
2,449,029 vertices, 61,859,140 edges, Chung-Lu alpha=0.8, 100-dim features)
run with the metric's model, 2-layer GCN [100, 256, 256], and 0.1% update
batches (61,859 updates: half hold-out inserts, half deletes of live edges).
configs[5] (the metric's own GCN/papers100M config) needs 8 GPUs; this is the
largest single-GPU configuration at the metric's model and batch fraction.

Arms
  (default)          our engine; `value` = device-timed throughput with the
                     batches already resident in HBM, `e2e` = the public
                     RTECEngine.step() API from pinned host buffers including
                     H2D of the batch and D2H of the per-update status/deltas.
  --impl reference   the reference's CPU path (the oracle port in oracle/, the
                     only place bench.py may execute it) on the same workload,
                     rank 0 only, on a bounded sample (see cpu_sample()).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events per step on the engine's stream, L2 flushed (256 MiB write)
between timed steps, max over ranks.  Multi-GPU (torchrun): the graph is
vertex-sharded over the ranks (owner = v mod N, paper_2603_20622_b200/shard.py)
and every batch runs once across all of them with one halo exchange per layer
over NCCL; total work is fixed as N grows (scaling "strong").
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge updates/sec and p50 batch latency, 2-layer GCN, 0.1% update batches"

WORKLOADS = {
    "c2-gcn": dict(desc="configs[1] graph (ogbn-products shape) with the metric's model: 2-layer GCN, 0.1% batches",
                   n=2449029, m=61859140, model="gcn", dims=[100, 256, 256], batch=61859, heads=1),
    "c2-sage": dict(desc="configs[1]: 2-layer GraphSAGE-mean, products shape, 0.1% batches",
                    n=2449029, m=61859140, model="graphsage", dims=[100, 256, 256], batch=61859, heads=1),
    "c1-gcn": dict(desc="configs[0]: 2-layer GCN 128 hidden, 100K/2M power-law, 1,000-update batches",
                   n=100000, m=2000000, model="gcn", dims=[128, 128, 128], batch=1000, heads=1),
    "c3-gat": dict(desc="configs[2]: 2-layer GAT, 4 heads, Reddit shape (232,965 V / 114.6M E, 602-dim), 0.1% batches",
                   n=232965, m=114615892, model="gat", dims=[602, 256, 256], batch=114616, heads=4),
    "c4-gin": dict(desc="configs[3]: 3-layer GIN (sum), R-MAT 10M V / 500M E, 128-dim, 0.1% batches",
                   n=10000000, m=500000000, model="gin", dims=[128, 128, 128, 128], batch=500000, heads=1,
                   gen="rmat"),
    "c4-gin-max": dict(desc="configs[3]: 3-layer GIN (max), R-MAT 10M V / 500M E, 128-dim, 0.1% batches",
                       n=10000000, m=500000000, model="gin_max", dims=[128, 128, 128, 128], batch=500000,
                       heads=1, gen="rmat"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2-gcn", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / cpu baseline)")
    ap.add_argument("--no-graphs", action="store_true", help="launch the per-batch pipeline eagerly (no CUDA graph)")
    ap.add_argument("--no-baselines", action="store_true", help="skip the UER / RTEC-Full GPU baseline batches")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-scale GPU-vs-CPU-port parity check")
    return ap.parse_args()


# ---------------------------------------------------------------- distributed
def dist_init():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # RTEC_BENCH_BACKEND=gloo: ranks may share one GPU (smoke runs of the sharded path on a 1-GPU box)
        if os.environ.get("RTEC_BENCH_BACKEND", "nccl") == "gloo":
            local = local % max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------- clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        if enabled:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            try:
                self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload
def make_workload(wl: dict, steps_total: int, device):
    """Graph on the GPU (bit-identical to the CPU generator), stream on the host."""
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features, rmat_edges

    gen = rmat_edges if wl.get("gen") == "rmat" else chung_lu_edges
    s, d = gen(wl["n"], wl["m"], seed=0, device=device)
    stream = UpdateStream(s, d, holdout=0.1, seed=0)
    batches = [stream.next_batch(wl["batch"]) for _ in range(steps_total)]
    X = features(wl["n"], wl["dims"][0], seed=1)
    return stream, batches, X


def algorithmic_bytes(name: str, wl: dict, layer_counters, n: int, prev_counters=None, fused: bool = False) -> float:
    """Algorithmic (compulsory) HBM bytes of one launch.

    layer_counters: [|E_curr|, |V_dst|, |S|, |R|, -, Σindeg(V_dst), -, layer] of the layer;
    prev_counters: the previous layer's (None for layer 0)."""
    e_curr, v_dst, n_src, _, _, sum_in = [float(x) for x in layer_counters[:6]]
    l = layer_counters[7]
    d_a = wl["dims"][int(l)]
    d_o = wl["dims"][int(l) + 1]
    f = 4.0
    if name == "aggregation":
        # in-run ids of V_dst + S-bitmap + δ rows once + S read/write + composed row write + list/offsets
        return 4 * sum_in + n / 8 + f * d_a * n_src + 3 * f * d_a * v_dst + 16 * v_dst
    if name == "k_gat_layer":
        # GAT (transform, then aggregate: rows of width d_o): in-run ids of V_dst + S-bitmap,
        # each gathered source row once (new Z rows, plus the logged old rows of S(l)),
        # S read + write, H write, DeltaLog write, el / er / ctx per head
        h = wl.get("heads", 1)
        new_rows = min(n, e_curr if layer_counters[3] == 0 else n)
        old_rows = min(n_src, e_curr)
        return (4 * sum_in + n / 8 + f * d_o * (new_rows + old_rows) + 4 * f * d_o * v_dst
                + 8 * h * (new_rows + old_rows) + 8 * h * v_dst)
    if name == "k_src_delta":
        # rows the kernel processes: all of S(l), or -- with the fused update epilogue writing
        # the δ rows of V_chg(l-1) -- only S(l) \ V_chg(l-1) = |S(l)| - |V_dst(l-1)|
        rows = n_src - (float(prev_counters[1]) if (fused and prev_counters is not None) else 0.0)
        return f * d_a * 3 * rows + 12 * rows
    if name in ("k_gemm_update", "k_gemm_tc"):
        # composed rows in (K padded to 32), H rows out (+ old H rows into the DeltaLog for
        # every layer but the last), 3xTF32 weight images
        last = int(l) == len(wl["dims"]) - 2
        kpad = (d_a + 31) // 32 * 32
        return f * kpad * v_dst + (1 if last else 3) * f * d_o * v_dst + 2 * f * kpad * d_o + 4 * v_dst
    if name == "k_expand":
        return 4 * e_curr + n / 8
    return 0.0


def apply_bytes(B: int, apply_ctr) -> float:
    """Algorithmic bytes of one batch_apply (SURVEY §8(d) "Structure"): the batch (op u8 +
    src/dst i32 + ts i64 = 17 B per update) read, the applied updates' ts (8 B), and the
    touched run suffixes moved by the merges: the old suffix + update items read and the
    new suffix written (out-runs 12 B per element with ts, in-runs 4 B), plus the in-place
    scratch staged and copied back."""
    w_out, s_out, w_in, s_in = [float(x) for x in apply_ctr]
    return 25.0 * B + 12.0 * (2 * w_out + 2 * s_out) + 4.0 * (2 * w_in + 2 * s_in)


def merge_bytes(apply_ctr) -> float:
    """Algorithmic bytes of the two run merges of one batch (both directions): the old
    suffix + update items read and the new suffix written, plus the in-place scratch staged
    and copied back (out-runs 12 B per element with ts, in-runs 4 B)."""
    w_out, s_out, w_in, s_in = [float(x) for x in apply_ctr]
    return 12.0 * (2 * w_out + 2 * s_out) + 4.0 * (2 * w_in + 2 * s_in)


def bench_config(args, wl: dict, world: int) -> dict:
    """The workload dict both arms print (same_config)."""
    sharded = world > 1
    return {"workload": args.workload, "desc": wl["desc"], "vertices": wl["n"], "edges": wl["m"],
            "model": wl["model"], "dims": wl["dims"], "batch_updates": wl["batch"],
            "batch_fraction": round(wl["batch"] / wl["m"], 6),
            "parallelism": f"vertex-sharded x{world} (owner = v mod {world}, owned + ghost rows, targeted "
                           "all-to-all of changed rows per layer)"
            if sharded else "single GPU",
            "l2": "flushed between timed steps (256 MiB write)"}


def gemm_flops(wl, layer_counters):
    l = int(layer_counters[7])
    return 2.0 * float(layer_counters[1]) * wl["dims"][l] * wl["dims"][l + 1]


# ---------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    import torch

    import paper_2603_20622_b200 as P
    from paper_2603_20622_b200 import _lib

    wl = WORKLOADS[args.workload]
    dev = torch.device("cuda", local)
    K, W = args.steps, args.warmup
    E2E = args.e2e_steps if args.e2e_steps is not None else min(K, 10)
    E2W = 2 if E2E else 0  # untimed warm-up calls of the public step() (pinned result buffers, allocator)
    PROF = min(K, 10)  # eager profiled pass after the timed region (per-kernel CUDA events)
    NB = 0 if (world > 1 or args.no_baselines) else 3  # batches per GPU baseline mode (UER, Full, NS)
    t0 = time.time()
    stream, batches, X = make_workload(wl, W + K + PROF + E2W + E2E + 3 * NB, dev)
    bs, bd, bt = stream.base()
    bundle = P.make_bundle(wl["model"], wl["dims"], heads=wl["heads"])
    sharded = world > 1
    if sharded:  # vertex-sharded over the ranks: one halo exchange per layer over NCCL
        from paper_2603_20622_b200.shard import Comm, ShardedRTECEngine

        eng = ShardedRTECEngine(bundle, wl["n"], tuple(torch.as_tensor(a, device=dev) for a in (bs, bd, bt)), X,
                                Comm(), max_batch=wl["batch"], reserve=max(1 << 20, wl["m"] // (2 * world)))
        g = eng.g
    else:
        g = P.DynamicGraph.from_tensors(wl["n"], torch.as_tensor(bs, device=dev), torch.as_tensor(bd, device=dev),
                                        torch.as_tensor(bt, device=dev), reserve=max(1 << 20, wl["m"] // 2))
        eng = P.RTECEngine(bundle, g, X, max_batch=wl["batch"], use_graphs=not args.no_graphs)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    lib = _lib.load()
    L = len(wl["dims"]) - 1
    # batches resident in HBM for the device-timed arm
    dev_batches = []
    for (op, s, d, t) in batches[: W + K + PROF]:
        dev_batches.append(tuple(torch.as_tensor(np.ascontiguousarray(a, dt), device=dev)
                                 for a, dt in ((op, np.uint8), (s, np.int32), (d, np.int32), (t, np.int64))))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    errs = torch.zeros(K + PROF, dtype=torch.int64, device=dev)
    ctrs = torch.zeros(PROF, L, 8, dtype=torch.int64, device=dev)
    actr = torch.zeros(PROF, 4, dtype=torch.int64, device=dev)
    bsz = []
    napp = torch.zeros(K, dtype=torch.int64, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]

    def run_step(i):
        """One batch from HBM-resident tensors; returns B.  Unsharded: enqueue only
        (no host sync inside the batch).  Sharded: step() synchronises for the
        error-word combine and the exchange counts."""
        op, s, d, t = dev_batches[i]
        if sharded:
            eng.step(op, s, d, t)
            return int(op.numel())
        B = g.stage(op, s, d, t)
        eng.enqueue_step(B)
        return B

    for i in range(W):
        run_step(i)
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local, enabled=not (args.no_clocks or args.profile))
    torch.cuda.synchronize()
    barrier(world)
    wall0 = time.time()
    total_updates = 0
    for k in range(K):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        evs[k][0].record()
        B = run_step(W + k)
        evs[k][1].record()
        total_updates += B
        errs[k : k + 1].copy_(eng.g.batch.err)  # (eng.g: a sharded engine may rebuild its shard graph)
        napp[k : k + 1].copy_(eng.g.batch.n_applied)
    torch.cuda.synchronize()
    barrier(world)
    wall = time.time() - wall0
    clk = clocks.stop()
    # per-kernel breakdown: PROF more batches, eager launches bracketed by CUDA events
    graphs_on = getattr(eng, "use_graphs", False)
    eng.use_graphs = False
    _lib.prof_enable(True)
    _lib.prof_report(reset=True)
    for k in range(PROF):
        flush.zero_()
        bsz.append(run_step(W + K + k))
        errs[K + k : K + k + 1].copy_(eng.g.batch.err)
        actr[k].copy_(eng.g.batch.apply_ctr)
        for l in range(L):
            ctrs[k, l].copy_(eng.fr[l].counters)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_report(reset=True)
    eng.use_graphs = graphs_on
    bad = [int(e) & _lib.ERR_OK for e in errs.cpu().tolist() if (int(e) & _lib.ERR_OK) != _lib.ERR_OK]
    if bad:
        raise RuntimeError(f"batch errors during timed run: {bad[:4]}")
    step_ms = [a.elapsed_time(b) for a, b in evs]
    applied = int(napp.sum().item())
    tot_s = sum(step_ms) / 1e3
    tot_s_max = max_over_ranks(tot_s, world)
    applied_all = sum_over_ranks(applied, world)
    value = applied_all / tot_s_max
    p50 = statistics.median(step_ms)
    p90 = float(np.percentile(step_ms, 90))
    # --- e2e through the public API from pinned host memory.  The long-lived objects built so far
    # (graph, engine, workload) move to the permanent GC generation, as a serving process would
    # after start-up, so a cyclic-GC pass does not walk them inside a timed call
    if os.environ.get("RTEC_BENCH_GC_FREEZE", "1") != "0":
        gc.collect()
        gc.freeze()
    e2e_ms, h2d, d2h = [], 0, 0
    e2e_upd = 0
    r = None
    for j in range(E2W):  # warm the public path (first-call allocations), untimed; each result stays
        op, s, d, t = batches[W + K + PROF + j]  # alive into the next call, as in the timed loop
        r = eng.step(*[torch.from_numpy(np.ascontiguousarray(a, dt)).pin_memory()
                       for a, dt in ((op, np.uint8), (s, np.int32), (d, np.int32), (t, np.int64))])
    torch.cuda.synchronize()
    for j in range(E2E):
        op, s, d, t = batches[W + K + PROF + E2W + j]
        hb = [torch.from_numpy(np.ascontiguousarray(a, dt)).pin_memory()
              for a, dt in ((op, np.uint8), (s, np.int32), (d, np.int32), (t, np.int64))]
        torch.cuda.synchronize()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record()
        r = eng.step(*hb)
        b_ev.record()
        torch.cuda.synchronize()
        e2e_ms.append(a_ev.elapsed_time(b_ev))
        e2e_upd += int(r.status.sum())
        h2d += sum(x.numel() * x.element_size() for x in hb)
        # RTECEngine._readback: status (B), 5 DegreeDelta columns (2B int32 each), err, n_delta, counters
        d2h += len(r.status) + 5 * 4 * 2 * len(r.status) + 8 + 8 + 64 * L
    e2e_val = None
    if E2E:
        e2e_s = max_over_ranks(sum(e2e_ms) / 1e3, world)
        e2e_val = sum_over_ranks(e2e_upd, world) / e2e_s
    # --- the paper's comparison set on the same GPU and stream: the same
    # public step() with the affected rows recomputed over full in-neighbourhoods (UER) and
    # every layer recomputed (RTEC-Full), and NS (fanout 10, approximate); per-batch time incl.
    # H2D / D2H like `e2e`.  NS runs last: it leaves the exact caches stale by design.
    baselines = {}
    for bi, mode in enumerate(("uer", "full", "ns")[: 3 if NB else 0]):
        ms, ups, acc = [], 0, 0
        for j in range(NB):
            op, s, d, t = batches[W + K + PROF + E2W + E2E + bi * NB + j]
            hb = [torch.from_numpy(np.ascontiguousarray(a, dt)).pin_memory()
                  for a, dt in ((op, np.uint8), (s, np.int32), (d, np.int32), (t, np.int64))]
            torch.cuda.synchronize()
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record()
            r = eng.step(*hb, mode=mode, fanout=10)
            b_ev.record()
            torch.cuda.synchronize()
            ms.append(a_ev.elapsed_time(b_ev))
            ups += int(r.status.sum())
            acc += sum(r.metrics.edge_accesses)
        baselines[mode] = {"p50_batch_ms": round(statistics.median(ms), 3),
                           "value": round(ups / (sum(ms) / 1e3), 1), "unit": "edge updates/s", "batches": NB,
                           "edge_accesses_per_batch": acc // NB}
    if baselines and e2e_ms:
        for mode in baselines:
            baselines[mode]["incremental_speedup"] = round(baselines[mode]["p50_batch_ms"] /
                                                           statistics.median(e2e_ms), 2)
    # --- roofline of the dominant kernel
    from_peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(from_peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if from_peaks else "fallback"
    C = ctrs.cpu().numpy()
    # the eager profiled pass: total of the bracketed library scopes (nested scopes excluded)
    nested = ("adj_merge", "k_expand", "k_agg_inc", "k_agg_inc_heavy", "k_hit_compact", "k_agg_sliced")
    prof_step_ms = sum(ms for name, (cnt, ms) in prof.items() if name not in nested)
    for l in range(L):
        C[:, l, 7] = l
    kernels = {}
    fused = bool(getattr(eng, "fused", False))
    AC = actr.cpu().numpy()
    for name, (cnt, ms) in prof.items():
        per_launch_ms = ms / max(cnt, 1)
        byts = 0.0
        if name in ("aggregation", "k_gat_layer", "k_src_delta", "k_gemm_update", "k_gemm_tc", "k_expand"):
            byts = sum(algorithmic_bytes(name, wl, C[k, l], wl["n"], C[k, l - 1] if l else None, fused)
                       for k in range(PROF) for l in range(L)) / max(cnt, 1)
        elif name == "batch_apply" and not sharded:
            byts = sum(apply_bytes(bsz[k], AC[k]) for k in range(PROF)) / max(cnt, 1)
        elif name == "adj_merge" and not sharded:
            byts = sum(merge_bytes(AC[k]) for k in range(PROF)) / max(cnt, 1)
        kernels[name] = {"launches": cnt, "total_ms": round(ms, 4), "ms_per_launch": round(per_launch_ms, 5),
                         "share": round(ms / max(prof_step_ms, 1e-9), 4),
                         "algo_GBps": round(byts / (per_launch_ms * 1e6), 1) if byts else None}
    if "aggregation" in kernels:
        kernels["aggregation"]["kernels"] = ("one scope per layer around the whole stage: k_agg_inc (light) + "
                                             "k_agg_inc_heavy (hub chunks), or k_hit_compact + k_agg_sliced passes")
    hot = [k for k in ("aggregation", "k_gat_layer", "k_gemm_tc", "k_gemm_update", "k_src_delta", "k_expand") if k in kernels]
    dom = max(hot, key=lambda k: kernels[k]["total_ms"]) if hot else None
    roof = None
    if dom:
        ach = kernels[dom]["algo_GBps"] or 0.0
        per_launch_bytes = ach * kernels[dom]["ms_per_launch"] * 1e6
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "peak_source": peak_src,
                "bytes_per_launch": per_launch_bytes, "traffic": None}
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            roof["traffic"] = json.load(open(tr)).get(args.workload, {}).get(dom)
        if roof["traffic"]:
            # the same launch against its measured DRAM traffic (ncu): how close the kernel runs to
            # the HBM roof for the bytes it actually moves (re-gathers included)
            dram = roof["traffic"] / (kernels[dom]["ms_per_launch"] * 1e6)
            roof["dram_achieved"] = round(dram, 1)
            roof["dram_frac"] = round(dram / hbm_peak, 4)
        if dom in ("k_gemm_update", "k_gemm_tc"):
            fl = sum(gemm_flops(wl, C[k, l]) for k in range(PROF) for l in range(L)) / max(kernels[dom]["launches"], 1)
            roof["tflops"] = round(fl / (kernels[dom]["ms_per_launch"] * 1e9), 2)
    res = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "edge updates/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(statistics.mean(step_ms), 4),
        "p50_batch_ms": round(p50, 4),
        "p90_batch_ms": round(p90, 4),
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded Chung-Lu graph, U(-1,1) features, make_bundle seed-0 weights)",
        "config": bench_config(args, wl, world),
        "e2e": {"value": round(e2e_val, 1) if e2e_val else None, "unit": "edge updates/s", "steps": E2E,
                "warmup": E2W,
                "h2d_bytes_per_step": h2d // max(E2E, 1), "d2h_bytes_per_step": d2h // max(E2E, 1),
                "p50_batch_ms": round(statistics.median(e2e_ms), 4) if e2e_ms else None,
                "batch_ms": [round(x, 3) for x in e2e_ms]},
        "gpu_launches": None,
        "roofline": roof,
        "gpu_baselines": baselines or None,
        "kernels": kernels,
        "frontier": {"e_curr": [int(np.mean(C[:, l, 0])) for l in range(L)],
                     "v_dst": [int(np.mean(C[:, l, 1])) for l in range(L)],
                     "n_src": [int(np.mean(C[:, l, 2])) for l in range(L)]},
        "clocks": clk,
        "setup_s": round(setup_s, 1),
        "wall_s": round(wall, 3),
    }
    nodes = getattr(eng, "graph_kernels", {}).get(wl["batch"])
    # captured step: every kernel node is one of ours; eager (sharded / --no-graphs): the scope count
    res["gpu_launches"] = (nodes if nodes and nodes > 0 else launches_per_step(prof, PROF)) * K
    res["cuda_graph"] = bool(graphs_on and nodes)
    res["graph_captures"] = len(getattr(eng, "_graphs", {}))
    res["compactions"] = int(getattr(eng.g, "compactions", 0))
    if sharded:  # per-rank exchange volume of the timed batches and the replica-free store
        import torch.distributed as dist

        xl = eng.exchange_log[W:W + K]
        mine = {"rank": rank, "exchange_rows_per_batch": sum(x["rows_sent"] for b in xl for x in b) / max(K, 1),
                "exchange_bytes_per_batch": sum(x["bytes_sent"] for b in xl for x in b) / max(K, 1),
                "exchange_rounds_per_batch": sum(x["rounds"] for b in xl for x in b) / max(K, 1),
                "admitted_ghosts_last_batch": int(eng.admitted)}
        mem = eng.memory_bytes()
        mine.update({k: v for k, v in mem.items() if k in ("n_own", "n_local", "cap")})
        mine["hbm_gb"] = round(sum(v for k, v in mem.items() if k not in ("n_own", "n_local", "cap")) / 1e9, 3)
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        res["shard"] = {"nranks": world, "backend": eng.comm.backend, "collective": "all_to_all_single",
                        "per_rank": allr}
    return res, eng.g, eng


def launches_per_step(prof, K):
    """Kernel launches of librtec per step (counted by the event hook's scopes)."""
    # scopes wrap single kernels except frontier_layer / batch_apply / adj_merge (multi-kernel);
    # count them from the static launch plan instead: see DESIGN.md §5 (launch census).
    n = 0
    for name, (cnt, _) in prof.items():
        n += cnt
    return int(round(n / max(K, 1)))


# ---------------------------------------------------------------- full-scale parity (GPU twin vs the CPU port)
def _rowwise(x, y):
    """(floored, strict) row-wise relative error (tests/helpers.py rowwise_rel / _strict)."""
    num = np.abs(x - y).max(axis=1)
    den = np.abs(y).max(axis=1)
    floored = float((num / np.maximum(den, max(1e-2 * float(den.max()), 1e-6))).max())
    nz = den > 0
    strict = float((num[nz] / den[nz]).max()) if nz.any() else 0.0
    zero_abs = float(num[~nz].max()) if (~nz).any() else 0.0
    return floored, strict, zero_abs


class GpuTwin:
    """A fresh GPU engine on the CPU leg's base graph that steps through the same batches;
    per batch the per-update status, DegreeDelta rows and frontier sizes must equal the
    C port's bit for bit, and after the last batch sampled rows of every H^l and S^l are
    compared (SURVEY §8(c) row-wise metric, fp32 vs f64) -- parity at the bench's own
    configuration, outside every timed region."""

    ROWS = 1 << 17

    def __init__(self, wl, bs, bd, bt, X):
        import torch

        import paper_2603_20622_b200 as P

        dev = torch.device("cuda", torch.cuda.current_device())
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
        self.g = P.DynamicGraph.from_tensors(wl["n"], t(bs), t(bd), t(bt), reserve=max(1 << 20, wl["m"] // 2))
        self.eng = P.RTECEngine(P.make_bundle(wl["model"], wl["dims"]), self.g, X, max_batch=wl["batch"])
        self.wl, self.batches, self.exact = wl, 0, True
        self.mismatch = []

    def step(self, batch, c_status, c_deltas, cport):
        r = self.eng.step(*batch)
        self.batches += 1
        ok = np.array_equal(r.status, c_status) and np.array_equal(r.deltas.astype(np.int64), c_deltas)
        for l in range(len(self.wl["dims"]) - 1):
            nv, ne = cport.frontier(l)
            ok = ok and (nv, ne) == (r.metrics.v_dst[l], r.metrics.e_curr[l])
        if not ok:
            self.mismatch.append(self.batches)
        self.exact = self.exact and ok

    def compare(self, cport) -> dict:
        import torch

        n = self.wl["n"]
        rng = np.random.default_rng(12345)
        indeg = self.g.in_deg[:n].cpu().numpy()
        ids = np.union1d(rng.choice(n, min(self.ROWS, n), replace=False), np.argsort(-indeg, kind="stable")[:1024])
        it = torch.as_tensor(ids, device=self.eng.dev)
        worst = {}
        L = len(self.wl["dims"]) - 1
        for kind, l in [("H", l) for l in range(1, L + 1)] + [("S", l) for l in range(L)]:
            mine = (self.eng.H[l] if kind == "H" else self.eng.S[l])[it].double().cpu().numpy()
            fl, st, za = _rowwise(mine, cport.rows(kind, l, ids))
            worst[f"{kind}{l}"] = {"rowwise_rel": fl, "strict_rel": st, "zero_rows_abs": za}
        return {"batches": self.batches, "rows": int(ids.size),
                "status_deltas_frontier_bit_exact": bool(self.exact), "mismatched_batches": self.mismatch,
                "max_rowwise_rel": max(v["rowwise_rel"] for v in worst.values()),
                "max_strict_rel": max(v["strict_rel"] for v in worst.values()), "tolerance": 1e-4,
                "per_tensor": worst,
                "against": "oracle/rtec_cpu.c f64 (C/OpenMP port of the oracle, pinned to the reference goldens)"}


# ---------------------------------------------------------------- reference (CPU) arm
def cpu_sample(wl_name: str, budget_s: float, max_steps: int, warmup: int = 1, twin: bool = False):
    """The reference's CPU path on the same workload: the C/OpenMP oracle port
    (oracle/rtec_cpu.c, pinned to the numpy oracle which is pinned to the
    reference), f64, every host thread.  Bounded sample: `warmup` untimed warm-up
    batches (at most 3: ~7 s each at c2), then timed batches until `budget_s` of
    CPU work or `max_steps`."""
    import os as _os

    from oracle import cport
    from oracle import models as OM
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features

    wl = WORKLOADS[wl_name]
    t0 = time.time()
    s, d = chung_lu_edges(wl["n"], wl["m"], seed=0)
    stream = UpdateStream(s, d, holdout=0.1, seed=0)
    bs, bd, bt = stream.base()
    b = OM.make_bundle(wl["model"], wl["dims"])
    W = [L["W"] for L in b.layers]
    W2 = [L["W2"] for L in b.layers] if wl["model"] == "gin" else None
    X = features(wl["n"], wl["dims"][0], 1)
    eng = cport.CPortEngine(wl["model"], wl["n"], bs, bd, bt, W, W2, wl["dims"], X.astype(np.float64),
                            degree_offset=b.degree_offset)
    setup = time.time() - t0
    tw = GpuTwin(wl, bs, bd, bt, X) if twin else None
    for _ in range(max(1, min(3, warmup))):  # untimed warm-up
        batch = stream.next_batch(wl["batch"])
        st, dl = eng.step(*batch)
        if tw:
            tw.step(batch, st, dl, eng)
    times, ups = [], 0
    while len(times) < max(1, max_steps):
        op, s1, d1, t1 = stream.next_batch(wl["batch"])
        t = time.time()
        st, dl = eng.step(op, s1, d1, t1)
        times.append(time.time() - t)
        ups += int(st.sum())
        if tw:
            tw.step((op, s1, d1, t1), st, dl, eng)
        if sum(times) > budget_s:
            break
    threads = eng.threads
    parity = tw.compare(eng) if tw else None
    eng.close()
    return {"value": ups / sum(times), "steps": len(times), "p50_s": statistics.median(times), "threads": threads,
            "setup_s": setup, "host_cpus": _os.cpu_count(), "parity": parity}


def main():
    args = parse()
    world, rank, local = dist_init()
    if args.impl == "reference":
        if rank != 0:
            return
        wl = args.workload
        wu = max(1, min(3, args.warmup))
        r = cpu_sample(wl, budget_s=150.0, max_steps=args.steps, warmup=wu)
        v = r["value"]
        out = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "edge updates/s", "n_gpus": world,
               "steps": r["steps"], "warmup": wu, "ms_per_step": round(r["p50_s"] * 1e3, 2),
               "p50_batch_ms": round(r["p50_s"] * 1e3, 2), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeded workload as the GPU arm)",
               "config": bench_config(args, WORKLOADS[wl], world), "setup_s": round(r["setup_s"], 1),
               "cpu_baseline": {"value": round(v, 1), "unit": "edge updates/s", "cores": r["threads"], "kind": "port",
                                "sample": f"{r['steps']} timed batches (after {wu} warm-up) of the {wl} workload, "
                                          f"C/OpenMP oracle port, f64, {r['threads']} threads of {r['host_cpus']} host CPUs"},
               "e2e": {"value": round(v, 1), "unit": "edge updates/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return
    res, g, eng = run_ours(args, world, rank, local)
    from oracle.cport import MODELS as PORT_MODELS

    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.profile) and \
            WORKLOADS[args.workload]["model"] in PORT_MODELS:
        del eng, g  # free HBM-side host references before the CPU run
        r = cpu_sample(args.workload, budget_s=30.0, max_steps=2, twin=not args.no_parity)
        res["parity"] = r["parity"]
        res["cpu_baseline"] = {"value": round(r["value"], 1), "unit": "edge updates/s", "cores": r["threads"],
                               "kind": "port",
                               "sample": f"{r['steps']} timed batch(es) after 1 warm-up of the same {args.workload} "
                                         f"workload: C/OpenMP oracle port (oracle/rtec_cpu.c), f64, {r['threads']} "
                                         f"threads of {r['host_cpus']} host CPUs; p50 {r['p50_s'] * 1e3:.0f} ms/batch"}
    if rank == 0:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
