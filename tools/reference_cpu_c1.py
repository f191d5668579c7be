"""The reference's own CPU path at configs[0] (C1), timed in the build container
(BASELINE.md §3 / SURVEY §8(d) "CPU baseline"): the GPU box has no /root/reference.

  CPU-full : reference DynamicGraph.apply_batch (graph.py:184) + reference_embeddings
             (models.py:487) of the post-batch graph -- the reference package itself, f64
  CPU-inc  : reference apply_batch + the oracle engine's incremental step (oracle/engine.py:
             Alg. 4 + Alg. 1 restated over numpy, f64)

C1: Chung-Lu 100K / 2M (seed 0, the bench's generator), GCN [128, 128, 128], one 1,000-update
batch.  Usage: OMP_NUM_THREADS=1 python tools/reference_cpu_c1.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from streamgnn import graph as RG  # noqa: E402
from streamgnn import models as RM  # noqa: E402

from oracle import models as OM  # noqa: E402
from oracle.engine import OracleEngine  # noqa: E402
from oracle.graph import OracleGraph  # noqa: E402
from paper_2603_20622_b200.workload import UpdateStream, chung_lu_edges, features  # noqa: E402

n, m, B, dims = 100_000, 2_000_000, 1000, [128, 128, 128]
out = {"config": "c1-gcn (configs[0]): Chung-Lu 100K / 2M, GCN [128,128,128], 1,000-update batch",
       "threads_env": os.environ.get("OMP_NUM_THREADS", "default"), "host_cpus": os.cpu_count()}
s, d = chung_lu_edges(n, m, seed=0)
stream = UpdateStream(s, d, holdout=0.1, seed=2)
bs, bd, bt = stream.base()
X = features(n, dims[0], seed=1).astype(np.float64)
op, s1, d1, t1 = stream.next_batch(B)

t = time.perf_counter()
rg = RG.DynamicGraph.from_edges(n, zip(bs.tolist(), bd.tolist(), bt.tolist()))
out["ref_from_edges_s"] = time.perf_counter() - t
batch = [RG.EdgeUpdate(RG.UpdateOp.INSERT if o == 0 else RG.UpdateOp.DELETE, int(a), int(b_), int(c))
         for o, a, b_, c in zip(op, s1, d1, t1)]
t = time.perf_counter()
res = rg.apply_batch(batch)
out["ref_apply_batch_s"] = time.perf_counter() - t
out["applied"] = len(res.applied)

bundle = RM.make_bundle("gcn", dims)
t = time.perf_counter()
H, A, C = RM.layer_embeddings(bundle, 0, rg, X)
out["ref_layer0_s"] = time.perf_counter() - t
t = time.perf_counter()
H2, A2, C2 = RM.layer_embeddings(bundle, 1, rg, H)
out["ref_layer1_s"] = time.perf_counter() - t
out["cpu_full_batch_s"] = out["ref_apply_batch_s"] + out["ref_layer0_s"] + out["ref_layer1_s"]
out["cpu_full_updates_per_s"] = out["applied"] / out["cpu_full_batch_s"]

og = OracleGraph.from_edges(n, bs, bd, bt)
oe = OracleEngine(OM.make_bundle("gcn", dims), og, X)
t = time.perf_counter()
o = oe.step(op, s1, d1, t1)
out["oracle_inc_step_s"] = time.perf_counter() - t
out["cpu_inc_batch_s"] = out["ref_apply_batch_s"] + out["oracle_inc_step_s"]
out["cpu_inc_updates_per_s"] = out["applied"] / out["cpu_inc_batch_s"]
# the oracle's incremental H^2 against the reference's full recompute of the same graph
num = np.abs(oe.H[2] - H2).max(axis=1)
den = np.maximum(np.abs(H2).max(axis=1), 1e-12)
out["oracle_vs_reference_strict_rel"] = float((num / den).max())
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
