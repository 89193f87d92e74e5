# whole-matrix L2 prefetch for small working sets (CSRK_MAT_PREFETCH=<MB>, 0 = off): C1 lines, parity subset
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_matpf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_matpf.log; tail -2 gpurun_out/pytest_matpf.log
for rep in 1 2; do
for cfg in "C1" "C1 --fp32"; do
  for pf in 0 96; do
    CSRK_MAT_PREFETCH=$pf timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', 'matpf=$pf', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/matpf_ab.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02e_C1_full python bench.py --config C1 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
