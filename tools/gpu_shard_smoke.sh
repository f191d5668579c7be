# sharded bench path smoke: 2 ranks sharing one B200 over gloo (collectives staged through host
# memory -- not a scaling number), c1-gcn and c2-gcn
mkdir -p gpurun_out
for w in c1-gcn c2-gcn; do
RTEC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --workload $w > gpurun_out/shard_smoke_$w.json 2> gpurun_out/shard_smoke_$w.err; echo "$w rc=$?"
tail -c 1500 gpurun_out/shard_smoke_$w.json
done
