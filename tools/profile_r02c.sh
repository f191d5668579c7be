# round-2 ncu evidence of HEAD (run under gpurun from the repo root; eager launches, one GPU)
#  - launch lists (per-launch durations) of one c2-gcn and one c3-gat batch
#  - --set full captures of the aggregation (light + hub passes, both layers), the tcgen05 update,
#    the GAT passes and the GAT projection -> DRAM bytes per launch for profiles/traffic.json
# The .ncu-rep files are exported to CSV on the box (raw metrics + details pages) and only the
# small ones are kept (gpurun copies back <= 64 MiB).
set -x
mkdir -p gpurun_out
B="python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02c_launches_c2gcn.csv $B > gpurun_out/r02c_list.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02c_launches_c3gat.csv $B --workload c3-gat > gpurun_out/r02c_list3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_agg_(light|heavy|batch)" -s 4 -c 4 -o gpurun_out/r02c_agg_c2 $B > gpurun_out/r02c_agg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 2 -c 2 -o gpurun_out/r02c_gemm_c2 $B > gpurun_out/r02c_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_src_delta -s 1 -c 2 -o gpurun_out/r02c_delta_c2 $B > gpurun_out/r02c_delta.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gat_(light|heavy)|k_gemm_tc" -s 6 -c 6 -o gpurun_out/r02c_gat_c3 $B --workload c3-gat > gpurun_out/r02c_gat.log 2>&1
for r in gpurun_out/r02c_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  sz=$(stat -c %s $r)
  if [ $sz -gt 12000000 ]; then rm -f $r; fi
done
gzip -f gpurun_out/r02c_*.raw.csv gpurun_out/r02c_*.details.csv gpurun_out/r02c_launches_*.csv
ls -la gpurun_out
