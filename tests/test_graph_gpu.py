"""GPU parity of the delta store (K1-K6) with the reference, through the C ABI.

Bit-exact against the golden fixtures produced by the reference itself and
against the oracle graph on larger random streams (graph.py:81-266).
"""

import numpy as np
import pytest

from helpers import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_20622_b200 as P

    return P


def _check_graph(g, esrc, edst, ets, indeg, outdeg):
    s, d, t = g.edges()
    assert np.array_equal(s, esrc) and np.array_equal(d, edst) and np.array_equal(t, ets)
    assert np.array_equal(g.in_degrees, indeg) and np.array_equal(g.out_degrees, outdeg)
    # in-adjacency mirrors out-adjacency (every live edge once in each)
    iv, iw = g.in_edges()
    o = np.lexsort((esrc, edst))
    assert np.array_equal(iv, edst[o]) and np.array_equal(iw, esrc[o])
    assert g.num_edges == esrc.size


def test_golden_graph_streams(P):
    z = golden("graph_streams.npz")
    for ci in range(3):
        n = int(z[f"c{ci}_n"])
        g = P.DynamicGraph.from_edges(n, (z[f"c{ci}_src"], z[f"c{ci}_dst"], z[f"c{ci}_ts"]))
        for b in range(int(z[f"c{ci}_nb"])):
            p = f"c{ci}_b{b}_"
            status, deltas = g.apply_arrays(z[p + "op"], z[p + "src"], z[p + "dst"], z[p + "ts"])
            assert np.array_equal(status, z[p + "status"]), (ci, b)
            assert np.array_equal(deltas, z[p + "deltas"]), (ci, b)
            _check_graph(g, z[p + "esrc"], z[p + "edst"], z[p + "ets"], z[p + "indeg"], z[p + "outdeg"])
            qin = np.concatenate([g.in_neighbors(int(v)) for v in z[p + "qv"]] + [np.zeros(0, np.int64)])
            qout = np.concatenate([g.out_neighbors(int(v)) for v in z[p + "qv"]] + [np.zeros(0, np.int64)])
            assert np.array_equal(qin, z[p + "qin"]) and np.array_equal(qout, z[p + "qout"])


def test_golden_errors_and_atomicity(P):
    z = golden("graph_streams.npz")
    names = [str(s) for s in z["err_names"]]
    g = P.DynamicGraph.from_edges(10, [(0, 1), (1, 2), (2, 3)])
    for i, name in enumerate(names):
        a = z[f"err{i}_batch"]
        before = g.edges()
        with pytest.raises(getattr(P, name)):
            g.apply_arrays(a[:, 0], a[:, 1], a[:, 2], a[:, 3])
        after = g.edges()
        assert all(np.array_equal(x, y) for x, y in zip(before, after))
        assert np.array_equal(g.in_degrees, np.bincount([1, 2, 3], minlength=10))


def test_object_api_matches_reference_shapes(P):
    g = P.DynamicGraph(6)
    U, I, D = P.EdgeUpdate, P.UpdateOp.INSERT, P.UpdateOp.DELETE
    r = g.apply_batch([U(I, 1, 2, 5), U(I, 3, 3, 6)])
    assert [u.ts for u in r.applied] == [5, 6] and r.rejected == ()
    assert r.deltas == (P.DegreeDelta(1, 0, 0, 0, 1), P.DegreeDelta(2, 0, 1, 0, 0), P.DegreeDelta(3, 0, 1, 0, 1))
    r = g.apply_batch([U(I, 1, 2, 7), U(D, 4, 5, 8)])
    assert r.applied == () and len(r.rejected) == 2 and r.deltas == ()
    assert g.has_edge(1, 2) and not g.has_edge(2, 1)
    with pytest.raises(P.InvalidVertex):
        g.in_neighbors(6)


def test_golden_coalesce(P):
    from paper_2603_20622_b200.graph import coalesce_arrays

    z = golden("coalesce.npz")
    for i in range(int(z["count"])):
        a = z[f"in{i}"]
        op, s, d, t = coalesce_arrays(a[:, 0], a[:, 1], a[:, 2], a[:, 3])
        got = np.stack([op.astype(np.int64), s, d, t], axis=1) if op.size else np.zeros((0, 4), np.int64)
        assert np.array_equal(got, z[f"out{i}"]), i


@pytest.mark.parametrize("B,reserve", [(300, None), (3000, None), (3000, 64)])
def test_random_stream_vs_oracle(P, B, reserve):
    """Mixed streams incl. rejects/self-loops, small and radix-sort batch sizes,
    and a tiny arena (forces relocation overflow -> compaction -> replay)."""
    _stream_vs_oracle(P, B, reserve, n=3000, m=40000)


@pytest.mark.parametrize("B", [800, 6000])
def test_long_runs_stream_vs_oracle(P, B):
    """~200 edges per vertex: the warp-per-chunk run merges (more than 96 slots per vertex),
    small update groups ranked by shuffles and hub groups of more than 32 updates by binary
    search; bit-exact against the oracle graph."""
    _stream_vs_oracle(P, B, None, n=600, m=120000)


def _stream_vs_oracle(P, B, reserve, n, m):
    from oracle.graph import OracleGraph
    from paper_2603_20622_b200.workload import chung_lu_edges

    rng = np.random.default_rng(B + (reserve or 0))
    s, d = chung_lu_edges(n, m, seed=7)
    ts = rng.permutation(m)
    g = P.DynamicGraph.from_edges(n, (s, d, ts), reserve=reserve)
    og = OracleGraph.from_edges(n, s, d, ts)
    for b in range(6):
        es, ed, _ = og.edges()
        k_del = B // 2
        pick = rng.choice(es.size, k_del, replace=False)
        ins = set()
        live = set(zip(es.tolist(), ed.tolist()))
        while len(ins) < B - k_del:
            a, c = int(rng.integers(n)), int(rng.integers(n))
            if rng.random() < 0.1:  # duplicate insert (rejected)
                j = int(rng.integers(es.size))
                a, c = int(es[j]), int(ed[j])
            if rng.random() < 0.05:
                c = a  # self-loop
            ins.add((a, c))
        ins -= set(zip(es[pick].tolist(), ed[pick].tolist()))
        ins = sorted(ins)
        op = np.array([1] * k_del + [0] * len(ins), np.uint8)
        bs = np.concatenate([es[pick], [x for x, _ in ins]]).astype(np.int64)
        bd = np.concatenate([ed[pick], [y for _, y in ins]]).astype(np.int64)
        # some absent deletes
        bs[:5], bd[:5] = rng.integers(n, size=5), rng.integers(n, size=5)
        keys = bs * n + bd
        _, first = np.unique(keys, return_index=True)
        keep = np.sort(first)
        op, bs, bd = op[keep], bs[keep], bd[keep]
        perm = rng.permutation(op.size)
        op, bs, bd = op[perm], bs[perm], bd[perm]
        bt = np.arange(op.size) + 10**6 * (b + 1)
        st, de = g.apply_arrays(op, bs, bd, bt)
        ost, ode = og.apply_batch(op, bs, bd, bt)
        assert np.array_equal(st, ost) and np.array_equal(de, ode), b
        es2, ed2, et2 = og.edges()
        _check_graph(g, es2, ed2, et2, og.in_deg, og.out_deg)


def test_deletion_round_trip_graph(P):
    from paper_2603_20622_b200.workload import chung_lu_edges

    s, d = chung_lu_edges(500, 5000, seed=2)
    g = P.DynamicGraph.from_edges(500, (s, d))
    e0 = g.edges()
    batch = [P.EdgeUpdate(P.UpdateOp.DELETE, int(a), int(b), 0) for a, b in zip(s[:50], d[:50])]
    batch += [P.EdgeUpdate(P.UpdateOp.INSERT, 499, v, 1) for v in range(30) if not g.has_edge(499, v)]
    g.apply_batch(batch)
    g.apply_batch(P.invert_batch(batch))
    e1 = g.edges()
    assert np.array_equal(e0[0], e1[0]) and np.array_equal(e0[1], e1[1])


def test_bulk_load_errors(P):
    with pytest.raises(P.InvalidVertex):
        P.DynamicGraph.from_edges(4, [(0, 1), (4, 0)])
    with pytest.raises(P.ConfigError):
        P.DynamicGraph.from_edges(4, [(0, 1), (0, 1)])
    with pytest.raises(P.ConfigError):
        P.DynamicGraph(1 << 31)
