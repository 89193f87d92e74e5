mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "long or pipeline or schedules or tile" > gpurun_out/pytest_pl3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pl3.log
tail -3 gpurun_out/pytest_pl3.log
timeout 600 python tools/powerlaw_probe.py 2000000 64 1000 20000 2>&1 | grep -v "^\[bench" > gpurun_out/pl3.txt
cat gpurun_out/pl3.txt
timeout 300 python tools/pl_one.py 20000 serial 0 2 2>&1 | grep plan
timeout 300 python tools/pl_one.py 1000 strided 4 2 2>&1 | grep plan
