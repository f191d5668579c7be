# Record of a reverted experiment (profiles/r02r_gemm_direct_epilogue_ab.md): the env knob it sets no longer exists at HEAD.
# A/B: staged vs direct (register) GEMM epilogue, and wide-N with direct + SA=3
mkdir -p gpurun_out
rm -f gpurun_out/ab_direct.txt
timeout 300 python -m pytest tests -m gpu -x -q -k "engine or gat or gin" > gpurun_out/ab_direct_pytest0.txt 2>&1; tail -2 gpurun_out/ab_direct_pytest0.txt >> gpurun_out/ab_direct.txt
RTEC_GEMM_DIRECT=1 timeout 300 python -m pytest tests -m gpu -x -q -k "engine or gat or gin" > gpurun_out/ab_direct_pytest1.txt 2>&1; tail -2 gpurun_out/ab_direct_pytest1.txt >> gpurun_out/ab_direct.txt
for w in c2-gcn c2-sage c3-gat c2-gcn; do
for cfg in "0 0" "1 0" "1 1"; do
  set -- $cfg
  RTEC_GEMM_DIRECT=$1 RTEC_GEMM_NWIDE=$2 timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_d_${w}_$1$2.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_d_${w}_$1$2.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w direct=$1 wide=$2', r['p50_batch_ms'], 'gemm', g('k_gemm_tc'))" >> gpurun_out/ab_direct.txt
done; done
cat gpurun_out/ab_direct.txt
