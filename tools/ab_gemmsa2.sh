mkdir -p gpurun_out
rm -f gpurun_out/ab_sa2.txt
for w in c2-gcn c2-gcn c2-sage; do
for a in 0 2; do
  RTEC_GEMM_SA=$a timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_sa2_${w}_$a.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_sa2_${w}_$a.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w sa=$a', r['p50_batch_ms'], 'gemm', g('k_gemm_tc'))" >> gpurun_out/ab_sa2.txt
done; done
cat gpurun_out/ab_sa2.txt
