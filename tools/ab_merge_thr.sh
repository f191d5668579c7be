# merge regime threshold 64 slots/vertex: which variant each workload now runs, and its timing
mkdir -p gpurun_out; out=gpurun_out/ab_mthr.txt; rm -f $out
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or merge or stream or apply" > gpurun_out/ab_mthr_pytest.txt 2>&1; tail -1 gpurun_out/ab_mthr_pytest.txt >> $out
for w in c4-gin c2-gcn c1-gcn c2-sage; do
for m in 1 0; do
  RTEC_MERGE_WARP=$m timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_mthr_${w}_$m.json 2>gpurun_out/ab_mthr_${w}_$m.err
  python -c "import json;r=json.load(open('gpurun_out/ab_mthr_${w}_$m.json'));k=r['kernels'];print('$w merge_warp=$m', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'apply', k['batch_apply']['ms_per_launch'], 'merge', k['adj_merge']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
