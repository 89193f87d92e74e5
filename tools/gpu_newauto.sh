# new auto schedule (tile 1536, 3-stage ring for regular rows, 3 / 4 CTAs) vs the round-1 auto (oldauto variant), interleaved; then GPU tests
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "C2" "C3" "C5" "C1" "C2 --fp32" "C3 --fp32" "C5 --fp32"; do
  for lib in default oldauto; do
    if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
    CSRK_LIB=$L timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', '$lib', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['config']['plan'], d['clocks']['sm_mhz'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/newauto_ab.txt
for lib in default oldauto; do
  if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
  echo "== powerlaw $lib"; CSRK_LIB=$L timeout 600 python tools/powerlaw_probe.py 2000000 1000 20000 2>&1 | tail -12
done 2>&1 | tee gpurun_out/newauto_powerlaw.txt
for lib in default oldauto; do
  if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
  CSRK_LIB=$L timeout 900 python bench.py --config C4 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('C4 $lib', d['config']['ms_per_iteration'], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], flush=True)"
done 2>&1 | tee -a gpurun_out/newauto_ab.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_newauto.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_newauto.log; tail -2 gpurun_out/pytest_newauto.log
