# plan re-sweep on the final kernel: C5 and C3 (tile x stages x CTAs/SM), fp64
mkdir -p gpurun_out
SWEEP_TILES=1536,2048,2560,3072 SWEEP_STAGES=2,3 SWEEP_CTAS=2,3 SWEEP_GATHER=0 SWEEP_DTYPES=float64 \
  timeout 1200 python tools/plan_sweep.py C5 C3 > gpurun_out/sweep_l.jsonl 2> gpurun_out/sweep_l.err; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/sweep_l.jsonl') if l.startswith('{')]
for cfg in ('C5','C3'):
    rs=sorted([r for r in rows if r['config']==cfg], key=lambda r: r['ms'])
    print(cfg)
    for r in rs[:8]: print('  ', r['variant'], r.get('nx'), 'T', r['tile_cost'], 'S', r['stages'], 'C', r['ctas'], r['ms'], r['gbs'], r['bitwise_equal'])
PY
