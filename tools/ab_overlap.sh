# A/B: apply results read back under the layer compute (RTEC_STEP_OVERLAP=1, default) vs after the step
mkdir -p gpurun_out; out=gpurun_out/ab_overlap.txt; rm -f $out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_overlap_pytest.txt 2>&1; tail -2 gpurun_out/ab_overlap_pytest.txt >> $out
for w in c2-sage c3-gat c1-gcn c2-gcn c2-sage c3-gat c1-gcn c2-gcn; do
for m in 1 0; do
  RTEC_STEP_OVERLAP=$m timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 10 > gpurun_out/ab_ov_${w}_$m.json 2>gpurun_out/ab_ov_${w}_$m.err
  python -c "import json;r=json.load(open('gpurun_out/ab_ov_${w}_$m.json'));print('$w overlap=$m', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], r['e2e']['batch_ms'])" >> $out 2>&1
done; done
cat $out
