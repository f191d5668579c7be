# c4-gin run merges: element-parallel (default regime for ~60 slots per vertex) vs warp-per-chunk
mkdir -p gpurun_out; out=gpurun_out/ab_mc4.txt; rm -f $out
for w in c4-gin c4-gin; do
for m in 1 2; do
  RTEC_MERGE_WARP=$m timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_mc4_${w}_$m.json 2>gpurun_out/ab_mc4_${w}_$m.err
  python -c "import json;r=json.load(open('gpurun_out/ab_mc4_${w}_$m.json'));k=r['kernels'];print('$w merge_warp=$m', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'apply', k['batch_apply']['ms_per_launch'], 'merge', k['adj_merge']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
