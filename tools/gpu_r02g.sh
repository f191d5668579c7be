# GAT bulk-copy row ring (RTEC_GAT_RING) and merge kernels (RTEC_MERGE_WARP): tests, then A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_engine_gpu.py tests/test_parity_configs_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/pytest_ring.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_ring.log
rm -f gpurun_out/ab_ring.txt
for cfg in "c3-gat 1 1" "c3-gat 0 1" "c3-gat 1 0" "c3-gat 1 1" "c3-gat 0 1" "c2-gcn 1 1" "c2-gcn 1 0" "c1-gcn 1 1" "c1-gcn 1 0" "c2-gcn 1 1" "c1-gcn 1 1"; do
  set -- $cfg
  RTEC_GAT_RING=$2 RTEC_MERGE_WARP=$3 timeout 300 python bench.py --workload $1 --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_ring_$1_$2_$3.json 2>gpurun_out/ab_ring_$1_$2_$3.err
  python -c "import json;r=json.load(open('gpurun_out/ab_ring_$1_$2_$3.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$1 ring=$2 merge_warp=$3', r['p50_batch_ms'], 'gat', g('k_gat_layer'), 'apply', g('batch_apply'), 'merge', g('adj_merge'))" >> gpurun_out/ab_ring.txt
done
cat gpurun_out/ab_ring.txt
