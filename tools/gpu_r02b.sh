# r02b: the multi-GPU C-ABI, cut-mode and fp32 tests, fp32 bench lines, the C1 plan sweep, the reference arm (C2, C1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dist.py tests/test_gpu_parity.py tests/test_abi.py tests/test_gpu_cg.py -x -q -m gpu > gpurun_out/pytest_r02b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02b.log
tail -3 gpurun_out/pytest_r02b.log
for cfg in "C2 --fp32" "C3 --fp32" "C5 --fp32" "C1 --fp32" "C3"; do
  timeout 300 python bench.py --config $cfg --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', d['ms_per_step'], d['roofline']['frac'], d['parity'], d['clocks']['sm_mhz'], flush=True)"
done 2>&1 | tee gpurun_out/f32_lines.txt
timeout 600 python bench.py --config C4 --fp32 --steps 5 --warmup 3 > gpurun_out/bench_C4f32.json 2> gpurun_out/bench_C4f32.err; echo "C4 f32 rc=$?"; head -c 700 gpurun_out/bench_C4f32.json; echo
bash tools/gpu_c1sweep.sh
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; echo "ref C2 rc=$?"; cat gpurun_out/bench_ref_C2.json
timeout 600 python bench.py --impl reference --config C1 > gpurun_out/bench_ref_C1.json 2> gpurun_out/bench_ref_C1.err; echo "ref C1 rc=$?"; cat gpurun_out/bench_ref_C1.json
