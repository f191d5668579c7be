# session re-entry check: GPU tests + smoke + default bench, hot-band A/B, c3-gat line
set -x
mkdir -p gpurun_out
bash tools/gpu_check.sh
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3"
rm -f gpurun_out/ab_hotband.txt
for mb in 0 64 128 0 64; do
  RTEC_HOT_MB=$mb timeout 300 $B > gpurun_out/ab_hotband_$mb.json 2>gpurun_out/ab_hotband_$mb.err
  python -c "import json;r=json.load(open('gpurun_out/ab_hotband_$mb.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('mb=$mb', r['p50_batch_ms'], g('k_agg_hot'), g('k_agg_inc'), g('k_agg_inc_heavy'), g('aggregation'))" >> gpurun_out/ab_hotband.txt
done
cat gpurun_out/ab_hotband.txt
timeout 600 python bench.py --workload c3-gat --steps 10 --no-cpu-baseline --no-parity > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c1-gcn --steps 20 --no-cpu-baseline --no-parity > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
echo done
