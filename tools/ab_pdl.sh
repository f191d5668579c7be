# A/B: programmatic dependent launch (RTEC_PDL=1, default) vs plain stream order
mkdir -p gpurun_out; out=gpurun_out/ab_pdl.txt; rm -f $out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pdl_pytest.txt 2>&1; tail -3 gpurun_out/ab_pdl_pytest.txt >> $out
for w in c1-gcn c2-gcn c2-sage c3-gat c1-gcn c2-gcn; do
for p in 1 0; do
  RTEC_PDL=$p timeout 400 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/ab_pdl_${w}_$p.json 2>gpurun_out/ab_pdl_${w}_$p.err
  python -c "import json;r=json.load(open('gpurun_out/ab_pdl_${w}_$p.json'));print('$w pdl=$p', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'])" >> $out 2>&1
done; done
cat $out
