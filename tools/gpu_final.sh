# end-of-session check of HEAD: GPU tests, smoke, default bench (CPU baseline + parity twin),
# the reference arm, other workloads, and the launch list of one c2-gcn batch
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/final_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "ref_rc=$?"
for w in c3-gat c1-gcn c2-sage c4-gin c4-gin-max; do
  timeout 900 python bench.py --workload $w --steps 20 --no-cpu-baseline --no-parity > gpurun_out/final_bench_$w.json 2>/dev/null; echo "$w rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final_launches_c2gcn.csv python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/final_list.log 2>&1
gzip -f gpurun_out/final_launches_c2gcn.csv
python - <<'PY'
import json, glob
for f in ['gpurun_out/final_bench.json'] + sorted(glob.glob('gpurun_out/final_bench_*.json')):
    try:
        r = json.load(open(f))
        print(f, r['config']['workload'], 'p50', r['p50_batch_ms'], 'value', r['value'], 'e2e', r['e2e']['value'],
              'frac', r['roofline']['frac'], 'clocks', r.get('clocks'), 'parity', (r.get('parity') or {}).get('max_strict_rel'))
    except Exception as e:
        print(f, 'ERR', e)
r = json.load(open('gpurun_out/final_reference.json')); print('reference', r.get('value'), r.get('cpu_baseline', {}).get('cores'))
PY
