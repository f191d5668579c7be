# Record of a reverted experiment (profiles/r02v_gat_unroll_ab.md): the env knob it sets no longer exists at HEAD.
# GAT recomputes: four rows in flight (RTEC_GAT_UNR4=1) vs two (0); old one-pair kernel for reference
mkdir -p gpurun_out; out=gpurun_out/ab_gatunr4.txt; rm -f $out
RTEC_GAT_UNR4=1 timeout 600 python -m pytest tests -m gpu -x -q -k "gat" > gpurun_out/ab_gatunr4_pytest.txt 2>&1; tail -1 gpurun_out/ab_gatunr4_pytest.txt >> $out
for w in c3-gat c3-gat c3-gat; do
for u in 1 0; do
  RTEC_GAT_UNR4=$u timeout 400 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/ab_gu4_${w}_$u.json 2>gpurun_out/ab_gu4_${w}_$u.err
  python -c "import json;r=json.load(open('gpurun_out/ab_gu4_${w}_$u.json'));k=r['kernels'];print('$w unr4=$u', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'gat', k['k_gat_layer']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
