mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdl.py -x -q -m gpu > gpurun_out/pytest_pdl.log 2>&1; echo "pytest pdl rc=$?"; tail -3 gpurun_out/pytest_pdl.log
bash tools/gpu_c5deep.sh
