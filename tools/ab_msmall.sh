# Record of a reverted experiment (profiles/r02w_merge_small_ab.md): the env knob it sets no longer exists at HEAD.
# A/B: small in-place run merges through shared memory (RTEC_MERGE_SMALL=1, default) vs scratch path
mkdir -p gpurun_out; out=gpurun_out/ab_msmall.txt; rm -f $out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_msmall_pytest.txt 2>&1; tail -2 gpurun_out/ab_msmall_pytest.txt >> $out
RTEC_MERGE_SMALL=1 RTEC_MERGE_WARP=2 timeout 600 python -m pytest tests -m gpu -x -q -k "graph or stream or merge or apply" > gpurun_out/ab_msmall_pytest_w2.txt 2>&1; tail -1 gpurun_out/ab_msmall_pytest_w2.txt >> $out
RTEC_MERGE_SMALL=1 RTEC_MERGE_WARP=0 timeout 600 python -m pytest tests -m gpu -x -q -k "graph or stream or merge or apply" > gpurun_out/ab_msmall_pytest_w0.txt 2>&1; tail -1 gpurun_out/ab_msmall_pytest_w0.txt >> $out
for w in c2-sage c3-gat c1-gcn c2-gcn c2-sage c3-gat c4-gin; do
for m in 1 0; do
  RTEC_MERGE_SMALL=$m timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 3 > gpurun_out/ab_ms_${w}_$m.json 2>gpurun_out/ab_ms_${w}_$m.err
  python -c "import json;r=json.load(open('gpurun_out/ab_ms_${w}_$m.json'));k=r['kernels'];print('$w small=$m', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'apply', k['batch_apply']['ms_per_launch'], 'merge', k['adj_merge']['ms_per_launch'])" >> $out 2>&1
done; done
cat $out
