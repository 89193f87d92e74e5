mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_long.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_long.log
tail -3 gpurun_out/pytest_long.log
timeout 900 python tools/powerlaw_probe.py 2000000 64 1000 20000 > gpurun_out/powerlaw2.txt 2>&1
grep -v "^\[bench" gpurun_out/powerlaw2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csrk_stream|long_rows_kernel" --csv \
  --log-file gpurun_out/pl_launches.csv python tools/powerlaw_probe.py 2000000 20000 > gpurun_out/pl_ncu.log 2>&1
python tools/launch_split.py gpurun_out/pl_launches.csv
