# tests, c3-gat + c2-gcn bench lines, launch list of one c3-gat batch (K13 on tcgen05)
set -x
NO_BENCH=1 bash tools/gpu_check.sh
timeout 600 python bench.py --workload c3-gat --steps 10 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c3gat.csv python bench.py --workload c3-gat --profile --no-graphs --no-baselines --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/ncu_c3.log 2>&1
echo done
