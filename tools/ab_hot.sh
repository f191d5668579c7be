# A/B of the L2 hot-row gather hint (RTEC_HOT_DEG) and the persisting carve-out (RTEC_PERSIST_MB), c2-gcn
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 3"
for cfg in "0 0" "90 0" "90 64" "60 96" "0 0" "150 48" "90 64"; do
  set -- $cfg
  RTEC_HOT_DEG=$1 RTEC_PERSIST_MB=$2 timeout 300 $B > gpurun_out/ab_hot_$1_$2.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_hot_$1_$2.json'));k=r['kernels'];print('hot=$1 persist=$2', r['p50_batch_ms'], k['k_agg_inc']['ms_per_launch'], k['k_agg_inc_heavy']['ms_per_launch'], k['aggregation']['ms_per_launch'])" >> gpurun_out/ab_hot.txt
done
cat gpurun_out/ab_hot.txt
