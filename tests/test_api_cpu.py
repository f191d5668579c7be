"""Host-side API checks that need no GPU: DynamicGraph constructor knobs
(graph.py:62-68 / pma.py:40-57 validation), edge-stream files, lossless checkpoint
edge tables, and from_reference on real reference bundles (when the reference is
importable in this container)."""

import os
import sys

import numpy as np
import pytest


def test_dynamic_graph_knob_validation():
    import paper_2603_20622_b200 as P

    for bad in ((0.0, 0.5), (0.5, 0.5), (0.3, 1.2)):
        with pytest.raises(P.ConfigError):
            P.DynamicGraph(10, density_bounds=bad)
    with pytest.raises(P.ConfigError):
        P.DynamicGraph(10, segment_slots=1)
    with pytest.raises(P.ConfigError):  # hi leaves no slack in the segment
        P.DynamicGraph(10, segment_slots=4, density_bounds=(0.25, 1.0))


def test_stream_file_round_trip(tmp_path):
    from paper_2603_20622_b200 import graph as G
    from paper_2603_20622_b200.errors import ConfigError

    ups = [G.EdgeUpdate(G.UpdateOp.INSERT, 1, 2, 3), G.EdgeUpdate(G.UpdateOp.DELETE, 4, 5, 2**60)]
    p = tmp_path / "s.txt"
    G.write_stream(str(p), ups)
    assert G.read_stream(str(p)) == ups
    p.write_text("# c\n\n+,1,2,3\n*,1,2,3\n")
    with pytest.raises(ConfigError, match=":4:"):
        G.read_stream(str(p))
    p.write_text("+,1,x,3\n")
    with pytest.raises(ConfigError, match="non-integer"):
        G.read_stream(str(p))


def test_checkpoint_edge_table_is_lossless():
    from paper_2603_20622_b200.formats import _edges_from_table, _edges_table

    ts = np.array([0, 1, 2**53 + 1, -(2**62) + 7, 2**63 - 1, -1], np.int64)
    src, dst = np.arange(6), np.arange(6)[::-1].copy()
    s, d, t = _edges_from_table(_edges_table(src, dst, ts))
    assert np.array_equal(s, src) and np.array_equal(d, dst) and np.array_equal(t, ts)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
@pytest.mark.parametrize("model", ["gcn", "graphsage", "gin", "gat", "pinsage", "monet", "commnet", "ggcn", "agnn"])
def test_from_reference_bundles(model):
    # a real reference OperatorBundle (models.py:364) adopted by value equals our seeded draws
    sys.path.insert(0, REF)
    try:
        from streamgnn import models as RM
    finally:
        sys.path.remove(REF)
    import paper_2603_20622_b200 as P

    for smoothing in ((True, False) if model == "gcn" else (True,)):
        ref = RM.make_bundle(model, [6, 5, 4], rng_seed=3, degree_smoothing=smoothing)
        ours = P.from_reference(ref)
        mine = P.make_bundle(model, [6, 5, 4], rng_seed=3, degree_smoothing=smoothing)
        assert ours.dims == mine.dims == tuple(ref.dims)
        assert ours.degree_offset == mine.degree_offset
        assert ours.agg_dims == mine.agg_dims == tuple(ref.agg_dims)
        for a, b, r in zip(ours.layers, mine.layers, ref.layers):
            for k in r.tensors:
                assert np.array_equal(a.tensors[k], r.tensors[k]) and np.array_equal(b.tensors[k], r.tensors[k]), k
            for k, v in r.scalars.items():
                if k != "degree_offset":
                    assert a.scalars[k] == v and b.scalars[k] == v, k
