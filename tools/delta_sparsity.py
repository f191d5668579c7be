"""Fraction of exact zeros in the layer-2 source deltas of c2-gcn (ReLU outputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_20622_b200 as P  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2-gcn"]
dev = torch.device("cuda", 0)
stream, batches, X = bench.make_workload(wl, 3, dev)
bs, bd, bt = stream.base()
g = P.DynamicGraph.from_tensors(wl["n"], torch.as_tensor(bs, device=dev), torch.as_tensor(bd, device=dev),
                                torch.as_tensor(bt, device=dev), reserve=max(1 << 20, wl["m"] // 2))
eng = P.RTECEngine(P.make_bundle(wl["model"], wl["dims"], heads=wl["heads"]), g, X, max_batch=wl["batch"])
for op, s, d, t in batches[:3]:
    eng.step(op, s, d, t)
torch.cuda.synchronize()
for l in range(1, eng.L):
    f = eng.fr[l]
    ns = int(f.n_src.item())
    rows = f.src_list[:ns].to(torch.int64)
    dl = eng.delta[l][rows]
    z = (dl == 0).float().mean().item()
    h = eng.H[l][rows]
    print(f"layer {l}: |S| {ns}, delta zero fraction {z:.3f}, H^{l} zero fraction {(h == 0).float().mean().item():.3f}")
    for w in (128, 64, 32):
        blk = (dl.reshape(ns, -1, w) == 0).all(dim=2).float().mean().item()
        print(f"   all-zero {w}-column blocks: {blk:.3f}")
