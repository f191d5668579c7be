# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (all ten models,
# hub chunking, forced compaction), plus memcheck of the same run with the captured CUDA graph
# (two-stream light / heavy passes).  Logs -> gpurun_out/sanitize_*.log, summary line per run.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c ': ok' gpurun_out/sanitize_$tool.log) models ok; $(tail -1 gpurun_out/sanitize_$tool.log)" | tee -a gpurun_out/sanitize_summary.txt
done
RTEC_SAN_GRAPHS=1 timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_memcheck_graphs.log 2>&1
echo "memcheck (CUDA graphs) rc=$? $(grep -c ': ok' gpurun_out/sanitize_memcheck_graphs.log) models ok; $(tail -1 gpurun_out/sanitize_memcheck_graphs.log)" | tee -a gpurun_out/sanitize_summary.txt
