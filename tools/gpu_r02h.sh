# cp.async GAT row ring (RTEC_GAT_RING=1): GAT parity tests with the ring on, then A/B on c3-gat
mkdir -p gpurun_out
RTEC_GAT_RING=1 timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_configs_gpu.py -q -x -k "gat" > gpurun_out/pytest_ring.log 2>&1; echo "pytest_ring_rc=$?"; tail -3 gpurun_out/pytest_ring.log
timeout 600 python -m pytest tests/test_graph_gpu.py -q -x > gpurun_out/pytest_graph.log 2>&1; echo "pytest_graph_rc=$?"; tail -2 gpurun_out/pytest_graph.log
rm -f gpurun_out/ab_ring2.txt
for r in 1 0 1 0; do
  RTEC_GAT_RING=$r timeout 300 python bench.py --workload c3-gat --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_ring2_$r.json 2>gpurun_out/ab_ring2_$r.err
  python -c "import json;r=json.load(open('gpurun_out/ab_ring2_$r.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('c3-gat ring=$r', r['p50_batch_ms'], 'gat', g('k_gat_layer'), 'apply', g('batch_apply'), 'merge', g('adj_merge'))" >> gpurun_out/ab_ring2.txt
done
for w in c2-gcn c1-gcn; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_merge2_$w.json 2>/dev/null; python -c "import json;r=json.load(open('gpurun_out/ab_merge2_$w.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w', r['p50_batch_ms'], 'apply', g('batch_apply'), 'merge', g('adj_merge'))" >> gpurun_out/ab_ring2.txt; done
cat gpurun_out/ab_ring2.txt
