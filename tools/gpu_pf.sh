# x prefetch into L2 (CSRK_X_PREFETCH=<MB limit>, 0 = off) A/B, then ncu full captures
mkdir -p gpurun_out
for cfg in "C1" "C5" "C1 --fp32" "C5 --fp32" "C3 --fp32" "C2 --fp32"; do
  for pf in 0 48 128; do
    CSRK_X_PREFETCH=$pf timeout 300 python bench.py --config $cfg --steps 50 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', 'pf=$pf', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], flush=True)"
  done
done 2>&1 | tee gpurun_out/pf_ab.txt
for c in "C5" "C2 --fp32" "C3" "C1"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02_${tag}_full python bench.py --config $c --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1
  echo "ncu $c rc=$?"
done
