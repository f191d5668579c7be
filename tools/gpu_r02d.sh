set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest_rc=$?"
tail -3 gpurun_out/pytest_gpu_full.log
bash tools/profile_r02c.sh
bash tools/sanitize.sh
