mkdir -p gpurun_out
timeout 900 python tools/check_gat_projection_precision.py > gpurun_out/gat_proj_precision.txt 2>&1; echo "prec_rc=$?"; cat gpurun_out/gat_proj_precision.txt | tail -4
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_configs_gpu.py -q -x -k "gat" > gpurun_out/pytest_fa.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_fa.log
rm -f gpurun_out/ab_fa.txt
for x in 1 0 1 0; do
  RTEC_GAT_FA=$x timeout 400 python bench.py --workload c3-gat --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_fa_$x.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_fa_$x.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('c3-gat fa=$x', r['p50_batch_ms'], 'gat', g('k_gat_layer'), 'delta', g('k_gat_delta'))" >> gpurun_out/ab_fa.txt
done
cat gpurun_out/ab_fa.txt
