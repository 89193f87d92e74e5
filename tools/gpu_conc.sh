mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_long.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_long.log
tail -3 gpurun_out/pytest_long.log
timeout 600 python tools/powerlaw_probe.py 2000000 64 1000 20000 2>&1 | grep -v "^\[bench" > gpurun_out/pl_conc.txt
cat gpurun_out/pl_conc.txt
