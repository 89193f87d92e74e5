# A/B: 32-bit-index gather address (default) vs __ldg(x + c) (CSRK_LDG_ASM=0 variant), interleaved
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r02c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02c.log; tail -2 gpurun_out/pytest_r02c.log
for rep in 1 2; do
for cfg in "C2" "C5" "C3" "C2 --fp32" "C3 --fp32"; do
  for lib in default noasm; do
    if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
    CSRK_LIB=$L timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', '$lib', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/asm_ab.txt
