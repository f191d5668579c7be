"""GPU parity of the vertex-sharded engine.

Two ranks share cuda:0 over a gloo group (the pool hands out one GPU; NCCL
refuses two ranks on one device, so the collectives are staged through host
memory -- the kernels, shards, global degrees and halo exchange are the same
code the NCCL path runs).  Every rank drives `ShardedRTECEngine` over the
same update stream; the parent process runs the unsharded engine and the
CPU oracle and compares:

- per-update status and DegreeDelta rows: bit-exact;
- V_dst(l) assembled over the shards and |E_curr(l)| summed: bit-exact;
- embeddings H^l assembled from the owners: within 1e-5 (row-wise; local-id
  summation order) of the unsharded engine and within 1e-4 of the oracle.
"""

import os
import socket
import tempfile

import numpy as np
import pytest

from helpers import rowwise_rel

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(cfg):
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features

    s, d = chung_lu_edges(cfg["n"], cfg["m"], seed=cfg["seed"])
    stream = UpdateStream(s, d, holdout=0.1, seed=cfg["seed"])
    X = features(cfg["n"], cfg["dims"][0], seed=cfg["seed"] + 1)
    batches = [stream.next_batch(cfg["B"]) for _ in range(cfg["nb"])]
    return stream.base(), X, batches


def _rank_main(rank, world, port, cfg, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    dev_i = rank if cfg.get("one_gpu_per_rank") else 0
    torch.cuda.set_device(dev_i)
    backend = cfg.get("backend", "gloo")
    kw = {"device_id": torch.device("cuda", dev_i)} if backend == "nccl" else {}
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world, **kw)
    import paper_2603_20622_b200 as P
    from paper_2603_20622_b200.shard import Comm, ShardedRTECEngine

    (bs, bd, bt), X, batches = _workload(cfg)
    b = P.make_bundle(cfg["model"], cfg["dims"], heads=cfg.get("heads", 1))
    eng = ShardedRTECEngine(b, cfg["n"], (bs, bd, bt), X, Comm(), max_batch=cfg["B"], reserve=cfg.get("reserve"),
                            ghost_headroom=cfg.get("headroom", 0.25), exchange_chunk=cfg.get("chunk", 1 << 20))
    res = {}
    # the store is not replicated: layer-input rows = owned + ghosts (+ headroom), never all n
    mem = eng.memory_bytes()
    res["n_local0"] = np.array([mem["n_local"], mem["cap"], mem["n_own"]])
    L = len(cfg["dims"]) - 1
    for i, (op, s, d, t) in enumerate(batches):
        r = eng.step(op, s, d, t)
        res[f"status{i}"], res[f"deltas{i}"] = r.status, r.deltas
        for l in range(L):
            res[f"vdst{i}_{l}"] = eng.frontier(l)[0]
            res[f"ecurr{i}_{l}"] = np.array(r.metrics.e_curr[l])
        res[f"sent{i}"] = np.array([x["rows_sent"] for x in eng.exchange_log[-1]] or [0])
        res[f"adm{i}"] = np.array([eng.admitted])
        if cfg.get("ckpt") and i == 0:  # per-rank checkpoint, then resume without a bootstrap
            ck = os.path.join(out_dir, "ck")
            eng.save(ck)
            dist.barrier()
            eng = ShardedRTECEngine.load(ck, Comm(), max_batch=cfg["B"])
    res["grown"] = np.array([getattr(eng, "grown", 0)])
    for l in range(L + 1):
        res[f"H{l}"] = eng.embeddings(l)
    ids = np.arange(0, cfg["n"], 7)
    res["query"] = eng.query(ids)
    if rank == 0:
        np.savez(os.path.join(out_dir, "shard.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def _run(cfg, world=2):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_20622_b200 as P
    from oracle import models as OM
    from oracle.engine import OracleEngine
    from oracle.graph import OracleGraph

    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), cfg, td), nprocs=world, join=True)
        sh = dict(np.load(os.path.join(td, "shard.npz")))
    (bs, bd, bt), X, batches = _workload(cfg)
    n, dims = cfg["n"], cfg["dims"]
    heads = cfg.get("heads", 1)
    eng = P.RTECEngine(P.make_bundle(cfg["model"], dims, heads=heads), P.DynamicGraph.from_edges(n, (bs, bd, bt)), X)
    oe = OracleEngine(OM.make_bundle(cfg["model"], dims, heads=heads), OracleGraph.from_edges(n, bs, bd, bt),
                      X.astype(np.float64))
    L = len(dims) - 1
    for i, (op, s, d, t) in enumerate(batches):
        r = eng.step(op, s, d, t)
        o = oe.step(op, s, d, t)
        assert np.array_equal(sh[f"status{i}"], r.status), i
        assert np.array_equal(sh[f"status{i}"], o["status"]), i
        assert np.array_equal(sh[f"deltas{i}"], o["deltas"]), i
        for l in range(L):
            assert np.array_equal(sh[f"vdst{i}_{l}"], o["frontier"][l]["vdst"]), (i, l)
            assert int(sh[f"ecurr{i}_{l}"]) == o["frontier"][l]["n_ecurr"], (i, l)
    for l in range(1, L + 1):
        # shards sum each in-run in LOCAL source-id order (owned ids, then ghosts): fp32
        # reassociation only, well inside the 1e-4 parity bound below
        assert rowwise_rel(sh[f"H{l}"], eng.embeddings(l)) <= 1e-5, l
        assert rowwise_rel(sh[f"H{l}"], oe.H[l]) <= 1e-4, l
    ids = np.arange(0, n, 7)
    assert np.array_equal(sh["query"], sh[f"H{L}"][ids])
    return sh


@pytest.mark.parametrize("model,dims", [("gcn", [32, 64, 32]), ("graphsage", [48, 64, 32]), ("gin", [32, 32, 32]),
                                        ("gat", [40, 32, 32]), ("gin_max", [32, 32, 32])])
def test_sharded_matches_unsharded(model, dims):
    _run(dict(model=model, dims=dims, n=3000, m=40000, B=300, nb=3, seed=21))


def test_sharded_three_layers_arena_replay():
    # tiny arena reserve: some rank runs out mid-stream, every rank replays the batch
    _run(dict(model="gcn", dims=[16, 16, 16, 16], n=2000, m=20000, B=400, nb=4, seed=22, reserve=64))


def test_sharded_gat_heads_three_ranks():
    # exchanged DeltaLog (GAT), several exchange rounds per layer
    _run(dict(model="gat", dims=[24, 64, 64], n=2500, m=30000, B=250, nb=2, seed=23, heads=4, chunk=97), world=3)


def test_sharded_fused_deltas_chunked_exchange():
    # fused source deltas written on receipt (GCN coefficients), exchange in rounds of 64 rows
    _run(dict(model="gcn", dims=[32, 64, 32], n=3000, m=40000, B=300, nb=3, seed=30, chunk=64), world=2)


def test_sharded_store_has_no_replicas():
    # rank 0's layer inputs hold its owned rows + ghosts, not all n vertices; rows are exchanged only
    # to peers (fewer than V_dst x (P - 1)); inserts admit new ghosts
    sh = _run(dict(model="graphsage", dims=[16, 32, 16], n=6000, m=9000, B=600, nb=3, seed=27), world=3)
    n_local, cap, n_own = sh["n_local0"].tolist()
    assert n_own == 2000 and n_local < 6000 and cap <= 6000
    assert sum(int(sh[f"adm{i}"][0]) for i in range(3)) > 0


def test_sharded_ghost_capacity_growth():
    # zero headroom: the first batches' admissions need a larger local id space (rebuild, ids kept)
    sh = _run(dict(model="gcn", dims=[16, 16, 16], n=20000, m=20000, B=1200, nb=3, seed=28, headroom=0.0))
    assert int(sh["grown"][0]) >= 1


def test_sharded_nccl_two_gpus():
    # the multi-GPU path proper: one rank per GPU over NCCL (device all_to_all / all_gather)
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(dict(model="gcn", dims=[32, 48, 32], n=3000, m=40000, B=300, nb=3, seed=29, backend="nccl",
              one_gpu_per_rank=True), world=2)


def test_sharded_nccl_single_rank():
    # one rank over NCCL: the device-tensor collective path the multi-GPU bench runs
    # (all_gather_into_tensor of ids / rows, uint8 MAX and int32 SUM all-reduces)
    _run(dict(model="gcn", dims=[32, 48, 32], n=3000, m=40000, B=300, nb=3, seed=24, backend="nccl"), world=1)


@pytest.mark.parametrize("model,heads", [("gcn", 1), ("gat", 2)])
def test_sharded_checkpoint_resume(model, heads):
    # each rank saves / restores its own shard between batches
    _run(dict(model=model, dims=[24, 32, 16], n=2500, m=30000, B=250, nb=3, seed=26, heads=heads, ckpt=True))
