mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
for w in c2-gcn c3-gat c1-gcn c2-sage c4-gin; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/b2_$w.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/b2_$w.json'));print('$w', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], r['value'], r['e2e']['value'], r['roofline']['frac'], (r.get('gpu_baselines') or {}).get('ns',{}).get('p50_batch_ms'))"
done
