"""The C/OpenMP oracle port (bench CPU baseline) agrees with the numpy oracle,
which is itself pinned to the reference (test_oracle_golden.py)."""

import numpy as np
import pytest

from helpers import rowwise_rel


@pytest.mark.parametrize("model,dims,smooth", [("gcn", [16, 24, 8], True), ("gcn", [8, 8, 8], False),
                                               ("graphsage", [12, 16, 8], True), ("gin", [8, 8, 8, 8], True)])
def test_cport_matches_oracle(model, dims, smooth):
    from oracle import cport
    from oracle import models as OM
    from oracle.engine import OracleEngine
    from oracle.graph import OracleGraph
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features

    n = 1500
    s, d = chung_lu_edges(n, 15000, seed=21)
    st = UpdateStream(s, d, 0.1, seed=2)
    bs, bd, bt = st.base()
    X = features(n, dims[0], seed=3).astype(np.float64)
    b = OM.make_bundle(model, dims, degree_smoothing=smooth)
    oe = OracleEngine(b, OracleGraph.from_edges(n, bs, bd, bt), X)
    W = [L["W"] for L in b.layers]
    W2 = [L["W2"] for L in b.layers] if model == "gin" else None
    ce = cport.CPortEngine(model, n, bs, bd, bt, W, W2, dims, X, degree_offset=b.degree_offset)
    for l in range(1, len(dims)):
        assert rowwise_rel(ce.H(l), oe.H[l]) <= 1e-10
    for _ in range(4):
        op, s1, d1, t1 = st.next_batch(120)
        # some rejects: duplicate insert of a live edge, absent delete
        op = np.concatenate([op, [0, 1]]).astype(np.uint8)
        s1 = np.concatenate([s1, [bs[0], 7]])
        d1 = np.concatenate([d1, [bd[0], 7 if (7, 7) not in set(zip(s1.tolist(), d1.tolist())) else 8]])
        t1 = np.concatenate([t1, [0, 0]])
        keys = s1 * n + d1
        _, first = np.unique(keys, return_index=True)
        keep = np.sort(first)
        op, s1, d1, t1 = op[keep], s1[keep], d1[keep], t1[keep]
        st_c, de_c = ce.step(op, s1, d1, t1)
        o = oe.step(op, s1, d1, t1)
        assert np.array_equal(st_c, o["status"]) and np.array_equal(de_c, o["deltas"])
        for l in range(len(dims) - 1):
            nv, ne = ce.frontier(l)
            assert nv == o["frontier"][l]["vdst"].size and ne == o["frontier"][l]["n_ecurr"]
        for l in range(1, len(dims)):
            assert rowwise_rel(ce.H(l), oe.H[l]) <= 1e-10, l


def test_cport_errors():
    from oracle import cport
    from oracle import models as OM

    b = OM.make_bundle("gcn", [4, 4])
    ce = cport.CPortEngine("gcn", 10, np.array([0, 1]), np.array([1, 2]), None, [b.layers[0]["W"]], None, [4, 4],
                           np.ones((10, 4)))
    with pytest.raises(ValueError, match="InvalidVertex"):
        ce.step(np.array([0, 0], np.uint8), np.array([1, 10]), np.array([3, 0]), np.zeros(2))
    with pytest.raises(ValueError, match="ConfigError"):
        ce.step(np.array([0, 0], np.uint8), np.array([1, 1]), np.array([3, 3]), np.zeros(2))
