# packed source-delta rows (RTEC_DELTA_PACK): tests, then A/B on the 256-wide workloads
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "packed" > gpurun_out/pytest_pack.log 2>&1; echo "pytest_pack_rc=$?"; tail -15 gpurun_out/pytest_pack.log
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_configs_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/pytest_pack2.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_pack2.log
rm -f gpurun_out/ab_pack.txt
for w in c2-gcn c2-sage c2-gcn c2-sage; do
for x in 1 0; do
  RTEC_DELTA_PACK=$x timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_pack_${w}_$x.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_pack_${w}_$x.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w pack=$x', r['p50_batch_ms'], 'light', g('k_agg_inc'), 'heavy', g('k_agg_inc_heavy'), 'stage', g('aggregation'), 'gemm', g('k_gemm_tc'))" >> gpurun_out/ab_pack.txt
done; done
cat gpurun_out/ab_pack.txt
