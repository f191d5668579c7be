"""C3-shape GAT parity (tests/test_parity_configs_gpu.py::test_c3_shape_gat) with the K13
projection on tcgen05 (3xTF32) and on the fp32 SIMT GEMM: worst row-wise errors vs the oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_20622_b200 as P  # noqa: E402
import test_parity_configs_gpu as T  # noqa: E402

for budget, name in ((8 << 30, "tcgen05 3xTF32 projection"), (0, "SIMT fp32 projection")):
    P.RTECEngine.GAT_IMG_BUDGET = budget
    os.environ["RTEC_PARITY_TAG"] = name
    if os.path.exists(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl")):
        os.remove(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"))
    T._stream_vs_oracle(P, "c3-gat-shape", "gat", [602, 256, 256], n=20000, m=2000000, B=2000, nb=4, seed=0, heads=4)
    for line in open(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl")):
        print(name, json.dumps(json.loads(line)["worst"]))
