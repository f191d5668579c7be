# GEMM bottleneck probe: remove B refills / A refills / splitting (wrong results, timing only)
mkdir -p gpurun_out
rm -f gpurun_out/ab_probe.txt
for w in c2-gcn c2-gcn; do
for p in 0 1 2 4 6 7; do
  RTEC_GEMM_PROBE=$p timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_p_${w}_$p.json 2>gpurun_out/ab_p_${w}_$p.err
  python -c "import json;r=json.load(open('gpurun_out/ab_p_${w}_$p.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w probe=$p', r['p50_batch_ms'], 'gemm', g('k_gemm_tc'))" >> gpurun_out/ab_probe.txt
done; done
cat gpurun_out/ab_probe.txt
