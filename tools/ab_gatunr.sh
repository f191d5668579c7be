# Record of a reverted experiment (profiles/r02v_gat_unroll_ab.md): the env knob it sets no longer exists at HEAD.
# A/B: GAT gathers with two row pairs in flight per warp (RTEC_GAT_UNR 24/25/26) vs one (0)
mkdir -p gpurun_out; out=gpurun_out/ab_gatunr.txt; rm -f $out
RTEC_GAT_UNR=42 timeout 600 python -m pytest tests -m gpu -x -q -k "gat" > gpurun_out/ab_gatunr_pytest.txt 2>&1; tail -2 gpurun_out/ab_gatunr_pytest.txt >> $out
for w in c3-gat c3-gat; do
for u in 0 24 33 42 43; do
  RTEC_GAT_UNR=$u timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_gu_${w}_$u.json 2>gpurun_out/ab_gu_${w}_$u.err
  python -c "import json;r=json.load(open('gpurun_out/ab_gu_${w}_$u.json'));k=r['kernels'];print('$w unr=$u', r['p50_batch_ms'], 'gat', k['k_gat_layer']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
