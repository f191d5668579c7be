mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_engine_gpu.py tests/test_heavy_order_gpu.py -q -x > gpurun_out/pytest_sort.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_sort.log
for w in c1-gcn c2-gcn c3-gat c1-gcn; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/b_$w.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/b_$w.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w', r['p50_batch_ms'], r['e2e']['p50_batch_ms'], 'apply', g('batch_apply'), 'merge', g('adj_merge'), 'launches', r['gpu_launches'])"
done
