mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csrk_stream|long_rows" -c 60 --csv --log-file gpurun_out/launches_C2_bench.csv \
  python bench.py --steps 20 --warmup 5 --cpu-budget 0.5 > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/launch_split.py gpurun_out/launches_C2_bench.csv | head
