"""Hub-chunk visit order is execution order only (layer.cu `plan_heavy`).

The heavy passes visit hub chunks sorted by relative run position (default,
RTEC_HEAVY_ORDER=1) or destination-major (0).  Partial rows are reduced in
chunk order either way, so every cached aggregate / embedding must be
bit-identical.  The switch is read once per process, hence one subprocess per
setting.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import paper_2603_20622_b200 as P
from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features
out = {}
for model, dims, heads in (("gat", [24, 64, 64], 4), ("gcn", [24, 32, 32], 1), ("gin_max", [16, 24, 16], 1)):
    n, m = 3000, 150000
    s, d = chung_lu_edges(n, m, seed=11)
    stream = UpdateStream(s, d, holdout=0.1, seed=11)
    bs, bd, bt = stream.base()
    g = P.DynamicGraph.from_edges(n, (bs, bd, bt))
    out[model + "_maxin"] = np.array(int(np.max(np.asarray(g.in_degrees))))
    eng = P.RTECEngine(P.make_bundle(model, dims, heads=heads), g, features(n, dims[0], seed=12))
    for _ in range(3):
        eng.step(*stream.next_batch(600))
    for l in range(len(dims) - 1):
        out[f"{model}_H{l + 1}"] = eng.embeddings(l + 1)
        out[f"{model}_A{l}"] = eng.aggregates(l)
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, order):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = str(tmp_path / f"order{order}.npz")
    env = dict(os.environ, RTEC_HEAVY_ORDER=str(order))
    subprocess.run([sys.executable, "-c", SCRIPT, path, ROOT], check=True, env=env, timeout=600)
    return np.load(path)


def test_heavy_order_bit_identical(tmp_path):
    a = _run(tmp_path, 1)
    b = _run(tmp_path, 0)
    for model in ("gat", "gcn", "gin_max"):
        assert int(a[model + "_maxin"]) > 2 * 512, "graph must have multi-chunk hubs"
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
