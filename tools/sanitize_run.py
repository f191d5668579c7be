"""Small incremental run of every model for compute-sanitizer (tools/sanitize.sh).

n = 8,000 / m = 240,000 Chung-Lu graph (hubs with in-runs > 512 edges, so the chunked
last-arrival reductions run), 3 mixed batches per model, eager launches (no CUDA graph),
plus the two-phase hot-band pass and a forced compaction (in-place merges + arena).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_20622_b200 as P  # noqa: E402
from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features  # noqa: E402

models = sys.argv[1:] or list(P.models.MODELS)
n, m = 8000, 240000
s, d = chung_lu_edges(n, m, seed=0)
for model in models:
    stream = UpdateStream(s, d, holdout=0.1, seed=3)
    bs, bd, bt = stream.base()
    heads = 4 if model == "gat" else 1
    dims = [64, 128, 64] if model != "gin" else [64, 128, 64, 64]
    g = P.DynamicGraph.from_edges(n, (bs, bd, bt), reserve=4096)
    X = features(n, dims[0], seed=1)
    graphs = os.environ.get("RTEC_SAN_GRAPHS", "0") == "1"
    eng = P.RTECEngine(P.make_bundle(model, dims, heads=heads), g, X, use_graphs=graphs)
    for k in range(3):
        op, s1, d1, t1 = stream.next_batch(600)
        r = eng.step(op, s1, d1, t1)
    eng.g.compact()
    op, s1, d1, t1 = stream.next_batch(600)
    eng.step(op, s1, d1, t1)
    torch.cuda.synchronize()
    H = eng.embeddings(len(dims) - 1)
    assert np.isfinite(H).all(), model
    print(f"{model}: ok, 4 batches, applied {int(r.status.sum())}", flush=True)
print("sanitize_run: all models done", flush=True)
