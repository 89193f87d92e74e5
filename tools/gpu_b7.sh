# serial batch 7 (rows of 7: no slot past the row end) vs 8, interleaved, C2 f64 / f32 and C4 CG
mkdir -p gpurun_out
for rep in 1 2 3; do
for cfg in "C2" "C2 --fp32"; do
  for sb in 8 7; do
    CSRK_SERIAL_BATCH=$sb timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', 'batch=$sb', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/b7_ab.txt
