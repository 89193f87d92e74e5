# C5 schedule after the instruction trims: gather mode x CTAs x tile (plan_sweep), serial batch 8 vs 4
mkdir -p gpurun_out
SWEEP_TILES=1536,2048,2560 SWEEP_STAGES=2 SWEEP_CTAS=2,3 SWEEP_GATHER=0,1 SWEEP_DTYPES=float64,float32 \
  timeout 900 python tools/plan_sweep.py C5 > gpurun_out/c5_sched.jsonl 2> gpurun_out/c5_sched.err; echo "sweep rc=$?"
CSRK_SERIAL_BATCH=4 SWEEP_TILES=1536,2048,2560 SWEEP_STAGES=2 SWEEP_CTAS=2,3 SWEEP_GATHER=0 SWEEP_DTYPES=float64,float32 \
  timeout 900 python tools/plan_sweep.py C5 > gpurun_out/c5_sched_b4.jsonl 2> gpurun_out/c5_sched_b4.err; echo "sweep b4 rc=$?"
python - <<'PY'
import json
for f in ('gpurun_out/c5_sched.jsonl','gpurun_out/c5_sched_b4.jsonl'):
    rows=[json.loads(l) for l in open(f) if l.startswith('{')]
    print(f)
    for r in sorted(rows, key=lambda r:(r['dtype'], r['ms'])):
        print('  ', r['dtype'], r['variant'], 'G', r['gather'], 'C', r['ctas'], 'T', r['tile_cost'], r['ms'], r['gbs'], r['bitwise_equal'])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02d_C2_full python bench.py --config C2 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/r02d_C5_full python bench.py --config C5 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
