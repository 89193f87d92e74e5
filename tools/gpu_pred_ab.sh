# A/B: predicated shared loads past the row end (default build) vs clamped loads (CSRK_PRED_LDS=0 variant)
mkdir -p gpurun_out
for cfg in "C5" "C2" "C3" "C5 --fp32" "C2 --fp32" "C3 --fp32" "C1"; do
  for lib in default nopred; do
    if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_nopred.so; fi
    CSRK_LIB=$L timeout 300 python bench.py --config $cfg --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', '$lib', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], flush=True)"
  done
done 2>&1 | tee gpurun_out/pred_ab.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02_C5pred_full python bench.py --config C5 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
