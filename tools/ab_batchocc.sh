mkdir -p gpurun_out
rm -f gpurun_out/ab_bocc.txt
for w in c2-gcn c4-gin c2-gcn; do
for o in 0 6; do
  RTEC_AGG_BATCH_OCC=$o timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_bocc_${w}_$o.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_bocc_${w}_$o.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w occ=$o', r['p50_batch_ms'], 'light', g('k_agg_inc'), 'stage', g('aggregation'))" >> gpurun_out/ab_bocc.txt
done; done
cat gpurun_out/ab_bocc.txt
