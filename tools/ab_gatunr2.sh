# GAT gathers: default (two row pairs in flight, 4 CTAs/SM) vs RTEC_GAT_UNR=1; full GPU suite first
mkdir -p gpurun_out; out=gpurun_out/ab_gatunr2.txt; rm -f $out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_gatunr2_pytest.txt 2>&1; tail -2 gpurun_out/ab_gatunr2_pytest.txt >> $out
for w in c3-gat c3-gat c3-gat; do
for u in 2 1; do
  RTEC_GAT_UNR=$u timeout 400 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/ab_gu2_${w}_$u.json 2>gpurun_out/ab_gu2_${w}_$u.err
  python -c "import json;r=json.load(open('gpurun_out/ab_gu2_${w}_$u.json'));k=r['kernels'];print('$w unr=$u', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'gat', k['k_gat_layer']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
