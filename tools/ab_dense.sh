# light-pass choice by hit density (RTEC_AGG_DENSE threshold; 0 = always one dst / warp, 2 = always batched)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -q -x -k "golden or oracle or edge" > gpurun_out/pytest_dense.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_dense.log
rm -f gpurun_out/ab_dense.txt
for w in c1-gcn c2-gcn c2-sage c4-gin c1-gcn c2-gcn; do
for t in 0.3 0 2; do
  RTEC_AGG_DENSE=$t timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_dense_${w}_$t.json 2>/dev/null
  python -c "import json;r=json.load(open('gpurun_out/ab_dense_${w}_$t.json'));k=r['kernels'];g=lambda n: k.get(n,{}).get('ms_per_launch');print('$w thr=$t', r['p50_batch_ms'], 'stage', g('aggregation'))" >> gpurun_out/ab_dense.txt
done; done
cat gpurun_out/ab_dense.txt
