mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "long or pipeline or schedules or tile" > gpurun_out/pytest_pl4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pl4.log
tail -2 gpurun_out/pytest_pl4.log
for e in "X=1" "CSRK_LONG_SERIAL=1"; do
  echo "== $e"
  env $e timeout 600 python tools/powerlaw_probe.py 2000000 1000 20000 2>&1 | grep -v "^\[bench"
done > gpurun_out/pl4.txt
cat gpurun_out/pl4.txt
SWEEP_DTYPES=float64 SWEEP_VARIANTS=strided SWEEP_NX=4,8 SWEEP_GATHER=2 SWEEP_CTAS=0 SWEEP_TILES=1152,1702,2048,2560 SWEEP_STAGES=2 \
  timeout 900 python tools/plan_sweep.py PL20000 2>/dev/null > gpurun_out/nx8.txt
python tools/sweep_table.py gpurun_out/nx8.txt
