# ncu evidence for the c3-gat bench step (run under gpurun from the repo root; eager launches)
set -x
B="python bench.py --workload c3-gat --profile --no-graphs --no-baselines --steps 1 --warmup 1 --e2e-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/gat_launches_order.csv $B > gpurun_out/gat_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gat_(light|heavy)" -s 4 -c 4 -o gpurun_out/gat_agg_order $B > gpurun_out/gat_agg.log 2>&1
ls -la gpurun_out
