# GPU check used during round 2: tests (new parity files first), smoke, default bench line.
# Run from the repo root under gpurun.  Outputs land in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
rm -f gpurun_out/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"
if [ -z "${NO_BENCH:-}" ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
fi
tail -3 gpurun_out/pytest_gpu.log
