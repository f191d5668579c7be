# round-2 ncu evidence for the c2-gcn bench step (run under gpurun from the repo root; eager launches)
set -x
B="python bench.py --profile --no-graphs --no-baselines --steps 1 --warmup 1 --e2e-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_c2gcn.csv $B > gpurun_out/r02_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_agg_light -s 4 -c 2 -o gpurun_out/r02_agg $B > gpurun_out/r02_agg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 2 -o gpurun_out/r02_gemm $B > gpurun_out/r02_gemm.log 2>&1
ls -la gpurun_out
