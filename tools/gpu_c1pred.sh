mkdir -p gpurun_out
for rep in 1 2 3; do
for cfg in "C1" "C1 --fp32"; do
  for lib in default noldgpred; do
    if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
    CSRK_LIB=$L timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', '$lib', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/c1pred_ab.txt
