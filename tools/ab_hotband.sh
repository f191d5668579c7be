# A/B of the two-phase hot-band aggregation (RTEC_HOT_MB), c2-gcn; plus its parity test
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -k "two_phase or golden_models" > gpurun_out/pytest_hot.log 2>&1; tail -2 gpurun_out/pytest_hot.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 3"
rm -f gpurun_out/ab_hotband.txt
for mb in 0 64 32 96 128 0 64; do
  RTEC_HOT_MB=$mb timeout 300 $B > gpurun_out/ab_hotband_$mb.json 2>gpurun_out/ab_hotband_$mb.err
  python -c "import json;r=json.load(open('gpurun_out/ab_hotband_$mb.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('mb=$mb', r['p50_batch_ms'], g('k_agg_hot'), g('k_agg_inc'), g('k_agg_inc_heavy'), g('aggregation'))" >> gpurun_out/ab_hotband.txt
done
cat gpurun_out/ab_hotband.txt
