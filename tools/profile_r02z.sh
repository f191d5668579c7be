# refresh the DRAM traffic of the dominant kernels at HEAD (profiles/traffic.json): c2-gcn aggregation
# passes, c2-gcn update GEMMs (+ tensor-pipe activity), c3-gat GAT passes; eager launches, one GPU
mkdir -p gpurun_out
B="python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none -k regex:"k_agg_(light|heavy|batch)" -s 4 -c 4 -o gpurun_out/r02z_agg_c2 $B > gpurun_out/r02z_agg.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_gemm_tc -s 2 -c 2 -o gpurun_out/r02z_gemm_c2 $B > gpurun_out/r02z_gemm.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_gat_(light|heavy)" -s 4 -c 4 -o gpurun_out/r02z_gat_c3 $B --workload c3-gat > gpurun_out/r02z_gat.log 2>&1
for r in gpurun_out/r02z_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  rm -f $r
done
gzip -f gpurun_out/r02z_*.raw.csv
ls -la gpurun_out/r02z*
