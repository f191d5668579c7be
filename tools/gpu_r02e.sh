set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_shard_gpu.py -q -x > gpurun_out/pytest_shard.log 2>&1; echo "shard_rc=$?"
tail -30 gpurun_out/pytest_shard.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest_rc=$?"
tail -3 gpurun_out/pytest_gpu_full.log
bash tools/sanitize.sh
bash tools/profile_r02c.sh
du -sh gpurun_out
