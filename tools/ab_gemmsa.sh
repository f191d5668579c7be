mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -q -x -k "golden" > gpurun_out/pytest_sa.log 2>&1; RTEC_GEMM_SA=4 timeout 600 python -m pytest tests/test_engine_gpu.py -q -x -k "golden" >> gpurun_out/pytest_sa.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_sa.log
rm -f gpurun_out/ab_sa.txt
for w in c2-gcn c2-gcn c3-gat; do
for a in 0 4; do
  RTEC_GEMM_SA=$a timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_sa_${w}_$a.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_sa_${w}_$a.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w sa=$a', r['p50_batch_ms'], 'gemm', g('k_gemm_tc'))" >> gpurun_out/ab_sa.txt
done; done
cat gpurun_out/ab_sa.txt
