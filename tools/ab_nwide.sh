# tcgen05 update GEMM: one N<=256 MMA per (K-step, product) (RTEC_GEMM_NWIDE=1) vs two N-halves (0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_configs_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/pytest_nwide.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_nwide.log
rm -f gpurun_out/ab_nwide.txt
for w in c2-gcn c3-gat c2-gcn c3-gat; do
for x in 1 0; do
  RTEC_GEMM_NWIDE=$x timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_nwide_${w}_$x.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_nwide_${w}_$x.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w nwide=$x', r['p50_batch_ms'], 'gemm', g('k_gemm_tc'), 'merge', g('adj_merge'), k.get('adj_merge',{}).get('algo_GBps'))" >> gpurun_out/ab_nwide.txt
done; done
cat gpurun_out/ab_nwide.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o gpurun_out/r02k_gemm_wide python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/r02k_gemm.log 2>&1
ncu -i gpurun_out/r02k_gemm_wide.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02k_gemm_wide.raw.csv.gz
