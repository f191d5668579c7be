"""Host-side logic of the vertex-sharded path with world_size 2
over gloo on CPU: the collectives `Comm` issues, the status-word combine, the
partition function, and the sharded frontier + halo exchange restated at set
level against the (unsharded) oracle engine's affected sets."""

import os
import socket
import tempfile

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as td:
        mp.spawn(fn, args=(world, _free_port(), td) + args, nprocs=world, join=True)
        return {f: dict(np.load(os.path.join(td, f))) for f in sorted(os.listdir(td))}


def _init(rank, world, port):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def _comm_main(rank, world, port, td):
    _init(rank, world, port)
    import torch
    import torch.distributed as dist

    from paper_2603_20622_b200.shard import Comm, combine_err_words

    c = Comm()
    assert c.staged and c.world == world and c.rank == rank
    ints = c.all_gather_ints([rank + 5, -1], torch.device("cpu"))
    # variable-length gather (DegreeDelta rows, frontier ids)
    var = c.all_gather_var(torch.arange(3 + rank, dtype=torch.int32) + 10 * rank, 2 + rank)
    # targeted exchange: rank r sends (r + 1) * (q + 1) rows of width 4 to rank q
    sc = torch.tensor([(rank + 1) * (q + 1) for q in range(world)], dtype=torch.int64)
    rc = c.all_to_all_counts(sc)
    rows = torch.cat([torch.full(((rank + 1) * (q + 1), 4), 100.0 * rank + q) for q in range(world)])
    got = c.all_to_all_rows(rows, sc.tolist(), rc.tolist())
    st = torch.tensor([rank, 1 - rank, 0], dtype=torch.uint8)
    c.all_reduce_(st, op=dist.ReduceOp.MAX)
    mine = (7 << 32) | 2 if rank == 0 else (3 << 32) | 8
    signed = mine - (1 << 64) if mine >= (1 << 63) else mine
    w = combine_err_words(c.all_gather_ints([signed], torch.device("cpu"))[:, 0])
    assert combine_err_words([-1, (5 << 32) | 1]) == (5 << 32) | 1  # all-ones (ok) never wins
    np.savez(os.path.join(td, f"r{rank}.npz"), ints=ints, var=var.numpy(), rc=rc.numpy(), got=got.numpy(),
             st=st.numpy(), w=np.array([w], np.uint64))
    dist.destroy_process_group()


def test_comm_collectives_gloo_world2():
    out = _spawn(_comm_main, 2)
    for r in (0, 1):
        z = out[f"r{r}.npz"]
        assert z["ints"].tolist() == [[5, -1], [6, -1]]
        assert z["var"].tolist() == [0, 1, 10, 11, 12]
        assert z["rc"].tolist() == [1 * (r + 1), 2 * (r + 1)]  # rank q sends (q + 1) * (r + 1) rows here
        g = z["got"]
        assert g.shape == ((r + 1) * 3, 4)
        assert (g[: r + 1] == 100.0 * 0 + r).all() and (g[r + 1:] == 100.0 * 1 + r).all()
        assert z["st"].tolist() == [1, 1, 0]
        assert int(z["w"][0]) == (3 << 32) | 8  # smallest position wins across ranks


def test_partition_covers_vertices_once():
    from paper_2603_20622_b200.shard import owner_of

    v = np.arange(1001)
    for P in (1, 2, 3, 8):
        own = owner_of(v, P)
        assert own.min() == 0 and own.max() == min(P, 1001) - 1
        assert sum((own == r).sum() for r in range(P)) == v.size


def _frontier_main(rank, world, port, td, n, m, B, nb, model):
    """Sharded F1 frontier: local edges (owned dst) + global Dg + exchanged V_chg."""
    _init(rank, world, port)
    import torch
    import torch.distributed as dist

    from oracle import models as OM
    from oracle.graph import OP_INSERT, OracleGraph
    from paper_2603_20622_b200.shard import Comm, owner_of
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges

    c = Comm()
    s, d = chung_lu_edges(n, m, seed=31)
    stream = UpdateStream(s, d, holdout=0.1, seed=31)
    bs, bd, bt = stream.base()
    g = OracleGraph.from_edges(n, bs, bd, bt)  # G_pre / G_post (global, for the shard filter)
    sdd = OM.make_bundle(model, [4, 4, 4]).src_degree_dependent
    res = {}
    for i in range(nb):
        op, s1, d1, t1 = stream.next_batch(B)
        old_out = g.out_deg.copy()
        status, _ = g.apply_batch(op, s1, d1, t1)
        ap = status.astype(bool)
        nn = np.uint64(n)
        es, ed = (g.out_keys // nn).astype(np.int64), (g.out_keys % nn).astype(np.int64)
        mine = owner_of(ed, world) == rank  # this rank's shard of G_post
        es, ed = es[mine], ed[mine]
        ins = ap & (op == OP_INSERT)
        loc_upd = ap & (owner_of(np.asarray(d1), world) == rank)
        is_ins = np.isin(es * n + ed, np.asarray(s1)[ins] * n + np.asarray(d1)[ins])
        # global Dg: each rank's local out-degree changes, summed (== rtec_shard_degrees)
        dloc = np.zeros(n, np.int64)
        np.add.at(dloc, np.asarray(s1)[loc_upd], np.where(op[loc_upd] == OP_INSERT, 1, -1))
        dg_t = torch.as_tensor(dloc)
        c.all_reduce_(dg_t)
        Dg = (dg_t.numpy() != 0) if sdd else np.zeros(n, bool)
        assert np.array_equal(Dg, (old_out != g.out_deg) if sdd else Dg)
        chg = np.zeros(n, bool)
        for l in range(2):
            S = Dg | chg
            vdst = np.zeros(n, bool)
            vdst[ed[S[es] & ~is_ins]] = True
            vdst[np.asarray(d1)[loc_upd]] = True
            assert not (vdst & (owner_of(np.arange(n), world) != rank)).any()  # only owned destinations
            # halo exchange: V_chg(l) = union of the shards' V_dst(l)
            t = torch.as_tensor(vdst.astype(np.int32))
            c.all_reduce_(t)
            chg = t.numpy() > 0
            res[f"v{i}_{l}"] = np.flatnonzero(chg)
    if rank == 0:
        np.savez(os.path.join(td, "f.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("model", ["gcn", "graphsage"])
def test_sharded_frontier_matches_oracle(model):
    from oracle import models as OM
    from oracle.engine import OracleEngine
    from oracle.graph import OracleGraph
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges

    n, m, B, nb = 1500, 12000, 120, 3
    out = _spawn(_frontier_main, 2, n, m, B, nb, model)["f.npz"]
    s, d = chung_lu_edges(n, m, seed=31)
    stream = UpdateStream(s, d, holdout=0.1, seed=31)
    bs, bd, bt = stream.base()
    X = np.zeros((n, 4))
    oe = OracleEngine(OM.make_bundle(model, [4, 4, 4]), OracleGraph.from_edges(n, bs, bd, bt), X)
    for i in range(nb):
        o = oe.step(*stream.next_batch(B))
        for l in range(2):
            assert np.array_equal(out[f"v{i}_{l}"], o["frontier"][l]["vdst"]), (model, i, l)


def _ghost_main(rank, world, port, td, n, m, B, nb):
    """The ghost-row protocol of shard.py / shard.cu restated at set level over gloo (world 3):
    load-time announce, admission by inserts (receiver and owner decide from the same batch),
    and the targeted exchange -- every rank holding an edge out of a changed vertex receives
    its row, and peers[u] has bit q exactly when rank q holds a ghost of u."""
    _init(rank, world, port)
    import torch

    from oracle.graph import OP_INSERT, OracleGraph
    from paper_2603_20622_b200.shard import Comm, owner_of
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges

    c = Comm()
    s, d = chung_lu_edges(n, m, seed=33)
    stream = UpdateStream(s, d, holdout=0.1, seed=33)
    bs, bd, bt = stream.base()
    g = OracleGraph.from_edges(n, bs, bd, bt)
    mine = owner_of(bd, world) == rank
    ghosts = set(np.unique(bs[mine][owner_of(bs[mine], world) != rank]).tolist())
    # announce: each ghost tells its owner (all_to_all of ids) -> peers bits of owned vertices
    out = [[u for u in sorted(ghosts) if owner_of(u, world) == q] for q in range(world)]
    sc = torch.tensor([len(x) for x in out], dtype=torch.int64)
    rc = c.all_to_all_counts(sc)
    ids = torch.tensor(sum(out, []) or [0], dtype=torch.int64)[: int(sc.sum())]
    got = c.all_to_all_rows(ids, sc.tolist(), rc.tolist()).tolist()
    src_rank = np.repeat(np.arange(world), rc.numpy())
    peers = {}
    for u, q in zip(got, src_rank.tolist()):
        peers[u] = peers.get(u, 0) | (1 << q)
    res = {}
    for i in range(nb):
        op, s1, d1, t1 = stream.next_batch(B)
        # admission: receiver admits sources of inserts into owned destinations; the owner
        # sets the peer bit for the same (source, rank) pairs
        for o, u, v in zip(op.tolist(), s1.tolist(), d1.tolist()):
            if o != OP_INSERT or owner_of(u, world) == owner_of(v, world):
                continue
            if owner_of(v, world) == rank:
                ghosts.add(u)
            if owner_of(u, world) == rank:
                peers[u] = peers.get(u, 0) | (1 << owner_of(v, world))
        g.apply_batch(op, s1, d1, t1)
        # a changed set (any vertex ids): every owned changed row goes to the ranks in peers
        chg = np.unique(np.concatenate([s1, d1]))
        sends = {q: sorted(u for u in chg.tolist() if owner_of(u, world) == rank and (peers.get(u, 0) >> q) & 1)
                 for q in range(world)}
        sc = torch.tensor([len(sends[q]) for q in range(world)], dtype=torch.int64)
        rc = c.all_to_all_counts(sc)
        ids = torch.tensor(sum((sends[q] for q in range(world)), []) or [0], dtype=torch.int64)[: int(sc.sum())]
        recv = set(c.all_to_all_rows(ids, sc.tolist(), rc.tolist()).tolist())
        nn = np.uint64(n)
        es, ed = (g.out_keys // nn).astype(np.int64), (g.out_keys % nn).astype(np.int64)
        here = owner_of(ed, world) == rank
        need = set(es[here][np.isin(es[here], chg) & (owner_of(es[here], world) != rank)].tolist())
        res[f"missing{i}"] = np.array(sorted(need - recv), np.int64)      # must be empty
        res[f"notghost{i}"] = np.array(sorted(recv - ghosts), np.int64)   # must be empty
        res[f"ghost_sources{i}"] = np.array(sorted(set(es[here][owner_of(es[here], world) != rank].tolist())
                                                   - ghosts), np.int64)   # must be empty
    # peers coherence: gather every rank's ghosts, compare with the owners' peer bits
    gl = c.all_gather_var(torch.tensor(sorted(ghosts) or [0], dtype=torch.int64)[: len(ghosts)], len(ghosts))
    cnt = c.all_gather_ints([len(ghosts)], torch.device("cpu"))[:, 0]
    holder = np.repeat(np.arange(world), cnt)
    want = {}
    for u, q in zip(gl.tolist(), holder.tolist()):
        if owner_of(u, world) == rank:
            want[u] = want.get(u, 0) | (1 << q)
    res["peers_ok"] = np.array([want == {u: b for u, b in peers.items() if b}], bool)
    np.savez(os.path.join(td, f"g{rank}.npz"), **res)
    import torch.distributed as dist

    dist.destroy_process_group()


def test_ghost_protocol_world3():
    out = _spawn(_ghost_main, 3, 2000, 16000, 300, 3)
    for r in range(3):
        z = out[f"g{r}.npz"]
        assert bool(z["peers_ok"][0]), r
        for i in range(3):
            assert z[f"missing{i}"].size == 0 and z[f"notghost{i}"].size == 0, (r, i)
            assert z[f"ghost_sources{i}"].size == 0, (r, i)
