# light-pass kernel for rows <= 128 floats: warp-batched (RTEC_AGG_BATCH=128, default) vs one
# destination per warp (RTEC_AGG_BATCH=0), on the narrow-row workloads
mkdir -p gpurun_out
rm -f gpurun_out/ab_batch.txt
for w in c1-gcn c2-sage c1-gcn c2-sage c2-gcn; do
for b in 128 0; do
  RTEC_AGG_BATCH=$b timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_batch_${w}_$b.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_batch_${w}_$b.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w batch=$b', r['p50_batch_ms'], 'light', g('k_agg_inc'), 'heavy', g('k_agg_inc_heavy'), 'stage', g('aggregation'))" >> gpurun_out/ab_batch.txt
done; done
cat gpurun_out/ab_batch.txt
