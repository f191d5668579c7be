# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (all models),
# plus the two-phase hot band.  Logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  RTEC_HOT_MB=1 timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py gcn graphsage > gpurun_out/sanitize_${tool}_hot.log 2>&1
  echo "$tool hot-band rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done
