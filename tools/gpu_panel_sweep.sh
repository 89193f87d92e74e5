# C5: streaming tiles vs column-sorted panels (capacity x consumer warps x CTAs/SM)
mkdir -p gpurun_out
TAG=${1:-r02p}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "panel" > gpurun_out/pytest_panel_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_panel_$TAG.log
tail -3 gpurun_out/pytest_panel_$TAG.log
OUT=gpurun_out/panel_sweep_$TAG.txt
: > $OUT
row() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['config']['plan'].get('n_panels'))"; }
for CFG in ${CFGS:-C5}; do
  CSRK_LAYOUT=0 timeout 300 python bench.py --config $CFG --steps 50 --cpu-budget 0.3 2>/dev/null | row "$CFG stream" >> $OUT
  for SPEC in ${SPECS:-"4096 8 2" "4096 16 1" "8192 16 1" "10240 16 1" "10240 8 1" "13312 16 1" "13312 8 1"}; do
    set -- $SPEC
    CSRK_LAYOUT=1 CSRK_PANEL_CAP=$1 CSRK_PANEL_WARPS=$2 CSRK_PANEL_CTAS=$3 timeout 300 python bench.py --config $CFG --steps 50 --cpu-budget 0.3 2>/dev/null | row "$CFG panels cap=$1 warps=$2 ctas=$3" >> $OUT
  done
done
cat $OUT
