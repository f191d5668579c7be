# c1-gcn launch list of HEAD (eager, serialised per-kernel durations) + full capture of the layer kernels
mkdir -p gpurun_out
B="python bench.py --workload c1-gcn --no-graphs --no-baselines --no-parity --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02u_launches_c1gcn.csv $B > gpurun_out/r02u_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_(light|heavy|batch)|k_gemm_tc|k_merge_items" -s 12 -c 8 -o gpurun_out/r02u_c1 $B > gpurun_out/r02u_full.log 2>&1
ncu -i gpurun_out/r02u_c1.ncu-rep --page raw --csv > gpurun_out/r02u_c1.raw.csv 2>/dev/null
gzip -f gpurun_out/r02u_c1.raw.csv gpurun_out/r02u_launches_c1gcn.csv
rm -f gpurun_out/r02u_c1.ncu-rep
ls -la gpurun_out | head
