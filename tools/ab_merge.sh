# merge kernels: warp-per-chunk (RTEC_MERGE_WARP=1, default) vs element-parallel (0); graph tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_engine_gpu.py tests/test_parity_configs_gpu.py -q -x > gpurun_out/pytest_merge.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_merge.log
rm -f gpurun_out/ab_merge.txt
for wl in c3-gat c2-gcn c1-gcn; do
for m in 1 0 1 0; do
  RTEC_MERGE_WARP=$m timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_merge_${wl}_$m.json 2>gpurun_out/ab_merge_${wl}_$m.err
  python -c "import json;r=json.load(open('gpurun_out/ab_merge_${wl}_$m.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$wl merge_warp=$m', r['p50_batch_ms'], 'apply', g('batch_apply'), 'merge', g('adj_merge'))" >> gpurun_out/ab_merge.txt
done; done
cat gpurun_out/ab_merge.txt
