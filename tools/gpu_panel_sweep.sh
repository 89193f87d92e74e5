# C5 (and C2/C3 for the record): streaming tiles vs column-sorted panels,
# panel capacity x CTAs per SM
mkdir -p gpurun_out
TAG=${1:-r02p}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "panel" > gpurun_out/pytest_panel_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_panel_$TAG.log
tail -3 gpurun_out/pytest_panel_$TAG.log
OUT=gpurun_out/panel_sweep_$TAG.txt
: > $OUT
for CFG in C5; do
  CSRK_LAYOUT=0 timeout 300 python bench.py --config $CFG --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG layout=stream', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'])" >> $OUT
  for CAP in 6144 8192 12288 16384 24576; do
    for CT in 1 2 3; do
      CSRK_LAYOUT=1 CSRK_PANEL_CAP=$CAP CSRK_PANEL_CTAS=$CT timeout 300 python bench.py --config $CFG --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG panels cap=$CAP ctas=$CT', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['config']['plan'])" >> $OUT
    done
  done
done
for CFG in C2 C3; do
  for L in 0 1; do
    CSRK_LAYOUT=$L timeout 300 python bench.py --config $CFG --steps 30 --cpu-budget 0.3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG layout=$L', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'])" >> $OUT
  done
done
cat $OUT
