# CG with p.Ap fused into the SpMV vs the separate dot kernel (C4 512^3, f64 / f32), CG tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q -m gpu > gpurun_out/pytest_cg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cg.log; tail -2 gpurun_out/pytest_cg.log
for prec in "" "--fp32"; do
  for mode in fused separate; do
    if [ $mode = separate ]; then export CSRK_NO_FUSED_DOT=1; else unset CSRK_NO_FUSED_DOT; fi
    timeout 900 python bench.py --config C4 $prec --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('C4 $prec', '$mode', d['ms_per_step'], d['config']['ms_per_iteration'], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
  done
done 2>&1 | tee gpurun_out/fused_dot_ab.txt
unset CSRK_NO_FUSED_DOT
