mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_engine_gpu.py tests/test_shard_gpu.py -q -x > gpurun_out/pytest_scan2.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_scan2.log
for w in c2-gcn c1-gcn c3-gat; do
  timeout 400 python bench.py --workload $w --steps 20 --no-cpu-baseline --no-parity --no-baselines > gpurun_out/bs_$w.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/bs_$w.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w', r['p50_batch_ms'], r['e2e']['p50_batch_ms'], r['e2e']['value'], 'apply', g('batch_apply'), 'frontier', g('frontier_layer'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_scan -c 200 --csv --log-file gpurun_out/scan_times.csv python bench.py --workload c2-gcn --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0 > /dev/null 2>&1
python -c "
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/scan_times.csv') if not l.startswith('=='))]
t=[float(r['Metric Value'])/1e3 for r in rows]
print('scan kernels', len(t), 'mean us %.2f'%(sum(t)/max(len(t),1)))
"
