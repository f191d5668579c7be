set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_shard_gpu.py -q > gpurun_out/pytest_shard.log 2>&1; echo "shard_rc=$?"; tail -30 gpurun_out/pytest_shard.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
B="python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_c1gcn.csv $B --workload c1-gcn > gpurun_out/r02f_list1.log 2>&1
gzip -f gpurun_out/r02f_launches_c1gcn.csv
python bench.py --workload c1-gcn --steps 20 --no-cpu-baseline --no-baselines --no-parity > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err
