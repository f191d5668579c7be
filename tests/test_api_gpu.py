"""Drop-in API surface beyond the incremental step (models.py:461-492;
linalg.py:17-60): RunResult.changed_final / Metrics.wall_time for every engine mode,
the GPU full-recompute functions under the reference's names, and NumericError."""

import numpy as np
import pytest

from helpers import rowwise_rel

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_20622_b200 as P

    return P


def _setup(P, model="gcn", dims=(16, 24, 8), n=1500, m=15000, seed=3, heads=1):
    from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features

    s, d = chung_lu_edges(n, m, seed=seed)
    stream = UpdateStream(s, d, holdout=0.1, seed=seed)
    bs, bd, bt = stream.base()
    X = features(n, dims[0], seed=seed + 1)
    return stream, (bs, bd, bt), X


@pytest.mark.parametrize("mode", ["inc", "uer", "full", "ns", "odec"])
def test_changed_final_and_wall_time(P, mode):
    stream, base, X = _setup(P)
    n = 1500
    eng = P.RTECEngine(P.make_bundle("gcn", [16, 24, 8]), P.DynamicGraph.from_edges(n, base), X)
    r = eng.step(*stream.next_batch(100), mode=mode)
    assert r.metrics.wall_time > 0
    cf = r.changed_final
    if mode == "full":
        assert np.array_equal(cf, np.arange(n))
    elif mode == "odec":
        assert cf.size == 0
    else:
        assert np.array_equal(cf, eng.frontier(1)[0])  # V_dst(L-1), ascending
        assert cf.size > 0 and np.all(np.diff(cf) > 0)


@pytest.mark.parametrize("model,dims,heads", [("gcn", [16, 24, 8], 1), ("graphsage", [16, 24, 8], 1),
                                              ("gin", [16, 16, 16], 1), ("gat", [16, 32, 32], 4)])
def test_reference_named_full_recompute(P, model, dims, heads):
    # models.py:461-492 names: layer_embeddings -> (H, A, C), forward_layer_reference,
    # reference_embeddings -- GPU full recompute vs the oracle's restatement
    from oracle import models as OM
    from oracle.graph import OracleGraph

    _, (bs, bd, bt), X = _setup(P, model, dims)
    n = 1500
    g = P.DynamicGraph.from_edges(n, (bs, bd, bt))
    ob = OM.make_bundle(model, dims, heads=heads)
    og = OracleGraph.from_edges(n, bs, bd, bt)
    b = P.make_bundle(model, dims, heads=heads)
    H1, A0, C0 = P.layer_embeddings(b, 0, g, X)
    rH1, rA0, rC0 = OM.layer_full(ob, 0, og, X.astype(np.float64))
    assert rowwise_rel(H1, rH1) <= TOL and rowwise_rel(A0, rA0) <= TOL
    assert np.allclose(C0.reshape(rC0.shape), rC0, rtol=1e-4, atol=1e-5)
    H2 = P.forward_layer_reference(b, g, H1, 1)
    assert rowwise_rel(H2, OM.layer_full(ob, 1, og, H1.astype(np.float64))[0]) <= TOL
    HL = P.reference_embeddings(b, g, X)
    assert rowwise_rel(HL, OM.reference_embeddings(ob, og, X.astype(np.float64))) <= TOL
    with pytest.raises(P.ConfigError):
        P.layer_embeddings(b, 0, g, X[:, :-1])


def test_numeric_error_gat_attention_overflow(P):
    # the reference raises on a non-finite exp / matvec (linalg.py:22-29, :55-60); here an
    # attention logit above ~88.7 overflows fp32 exp -> NumericError at bootstrap
    _, base, X = _setup(P, "gat", (8, 8, 8))
    b = P.make_bundle("gat", [8, 8, 8])
    big = [P.LayerWeights(w.in_dim, w.out_dim, {"W": w.tensors["W"], "a": np.asarray(w.tensors["a"]) * 1e4})
           for w in b.layers]
    hot = P.make_bundle("gat", [8, 8, 8], weights=big)
    with pytest.raises(P.NumericError):
        P.RTECEngine(hot, P.DynamicGraph.from_edges(1500, base), X)


def test_numeric_error_non_finite_update(P):
    # a non-finite feature reaches the update matvec once an edge from it is inserted
    stream, (bs, bd, bt), X = _setup(P, "gcn", (8, 8, 8))
    n = 1500
    outdeg = np.bincount(bs, minlength=n)
    u = int(np.flatnonzero(outdeg == 0)[0])
    X = X.copy()
    X[u, 3] = np.inf
    eng = P.RTECEngine(P.make_bundle("gcn", [8, 8, 8]), P.DynamicGraph.from_edges(n, (bs, bd, bt)), X)
    eng.step(*stream.next_batch(50))  # finite so far
    with pytest.raises(P.NumericError):
        eng.step(np.zeros(1, np.uint8), np.array([u]), np.array([(u + 1) % n]), np.array([7]))
    with pytest.raises(P.NumericError):  # and at bootstrap when the source already has edges
        P.RTECEngine(P.make_bundle("gcn", [8, 8, 8]),
                     P.DynamicGraph.from_edges(n, (np.append(bs, u), np.append(bd, (u + 1) % n))), X)
