# A/B: column-slice passes of the c2-gcn aggregation (RTEC_AGG_SLICE, 0 = whole rows) and the
# light-pass kernel choice for 128-wide slices (RTEC_AGG_BATCH=0: one destination per warp)
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3"
rm -f gpurun_out/ab_slice.txt
for cfg in "0 128" "128 128" "128 0" "0 128" "128 128"; do
  set -- $cfg
  RTEC_AGG_SLICE=$1 RTEC_AGG_BATCH=$2 timeout 300 $B > gpurun_out/ab_slice_$1_$2.json 2>gpurun_out/ab_slice_$1_$2.err
  python -c "import json;r=json.load(open('gpurun_out/ab_slice_$1_$2.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('slice=$1 batch=$2', r['p50_batch_ms'], g('k_agg_inc'), g('k_agg_inc_heavy'), g('aggregation'))" >> gpurun_out/ab_slice.txt
done
cat gpurun_out/ab_slice.txt
