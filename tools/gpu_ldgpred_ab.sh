# A/B: predicated x gathers per batch (one asm block, default) vs unpredicated (x[0] for spare lanes)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_ldg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ldg.log; tail -2 gpurun_out/pytest_ldg.log
for rep in 1 2; do
for cfg in "C5" "C2" "C3" "C1" "C5 --fp32" "C2 --fp32" "C3 --fp32"; do
  for lib in default noldgpred; do
    if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
    CSRK_LIB=$L timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', '$lib', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/ldgpred_ab.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02j_C5_full python bench.py --config C5 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r02j_C5_full.ncu-rep > gpurun_out/r02j_C5_stream_ncu_full.txt 2>&1
ncu -i gpurun_out/r02j_C5_full.ncu-rep --page raw --csv > gpurun_out/r02j_C5_raw.csv 2>/dev/null
rm -f gpurun_out/r02j_C5_full.ncu-rep
