# x prefetch into L2 (CSRK_X_PREFETCH=<MB limit>, 0 = off): C1, C5, C3 and fp32 lines
mkdir -p gpurun_out
for cfg in "C1" "C5" "C1 --fp32" "C5 --fp32" "C3 --fp32" "C3"; do
  for pf in 0 48 128; do
    CSRK_X_PREFETCH=$pf timeout 300 python bench.py --config $cfg --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', 'pf=$pf', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'])" 
  done
done
