# source-level instruction hot spots of the c2-gcn layer-1 warp-batched aggregation (k_agg_batch)
mkdir -p gpurun_out
B="python bench.py --profile --no-graphs --no-baselines --no-parity --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_batch" -s 1 -c 1 -o gpurun_out/r02y_aggbatch $B > gpurun_out/r02y.log 2>&1
ncu -i gpurun_out/r02y_aggbatch.ncu-rep --page source --csv --print-source sass > gpurun_out/r02y_aggbatch.sass.csv 2>/dev/null
ncu -i gpurun_out/r02y_aggbatch.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02y_aggbatch.cuda.csv 2>/dev/null
ncu -i gpurun_out/r02y_aggbatch.ncu-rep --page raw --csv > gpurun_out/r02y_aggbatch.raw.csv 2>/dev/null
gzip -f gpurun_out/r02y_aggbatch.*.csv
ls -la gpurun_out/r02y*
rm -f gpurun_out/r02y_aggbatch.ncu-rep
