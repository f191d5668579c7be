# sharded bench path smoke (2 ranks on one GPU over gloo) + default bench lines of HEAD
mkdir -p gpurun_out
RTEC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload c1-gcn --steps 3 --warmup 3 > gpurun_out/bench_shard2_c1.json 2> gpurun_out/bench_shard2_c1.err; echo "shard_bench_rc=$?"
tail -c 1500 gpurun_out/bench_shard2_c1.json; tail -5 gpurun_out/bench_shard2_c1.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
timeout 600 python bench.py --workload c3-gat --steps 10 --no-cpu-baseline --no-parity > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c1-gcn --steps 20 --no-cpu-baseline --no-parity > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python - <<'PY'
import json
for f in ['gpurun_out/bench.json','gpurun_out/bench_c3.json','gpurun_out/bench_c1.json']:
    try:
        r=json.load(open(f)); print(f, r['p50_batch_ms'], r['value'], r['e2e']['value'], r['roofline']['frac'], r.get('clocks'))
    except Exception as e: print(f, 'ERR', e)
PY
