mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r01c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r01c.log
tail -3 gpurun_out/pytest_r01c.log
bash tools/gpu_dist1.sh r01c
