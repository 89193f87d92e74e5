# serial batch 16 (C5: one gather round trip for rows up to 16) vs 8, interleaved
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "C5" "C5 --fp32" "C2"; do
  for sb in 8 16; do
    CSRK_SERIAL_BATCH=$sb timeout 300 python bench.py --config $cfg --steps 100 --cpu-budget 0.3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg', 'batch=$sb', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
  done
done
done 2>&1 | tee gpurun_out/b16_ab.txt
CSRK_SERIAL_BATCH=16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02i_C5b16_full python bench.py --config C5 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r02i_C5b16_full.ncu-rep > gpurun_out/r02i_C5b16_stream_ncu_full.txt 2>&1
ncu -i gpurun_out/r02i_C5b16_full.ncu-rep --page raw --csv > gpurun_out/r02i_C5b16_raw.csv 2>/dev/null
rm -f gpurun_out/r02i_C5b16_full.ncu-rep
