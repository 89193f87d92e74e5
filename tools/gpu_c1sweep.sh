# small-matrix plan sweep (C1, L2 flushed before every launch): tile x stages x CTAs/SM
mkdir -p gpurun_out
SWEEP_FLUSH=1 SWEEP_TILES=512,768,1024,1536,2048 SWEEP_STAGES=2,3,4 SWEEP_CTAS=2,3,4,6 SWEEP_DTYPES=float64,float32 SWEEP_GATHER=0 \
  timeout 1200 python tools/plan_sweep.py C1 > gpurun_out/c1_sweep.jsonl 2> gpurun_out/c1_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/c1_sweep.jsonl') if l.startswith('{')]
for dt in ('float64','float32'):
    rs=sorted([r for r in rows if r['dtype']==dt], key=lambda r: r['ms'])
    print(dt, 'best 8:')
    for r in rs[:8]: print('  ', r['tile_cost'], r['stages'], r['ctas'], r['ms'], r['gbs'], r['bitwise_equal'])
    d=[r for r in rs if r['tile_cost']==2048 and r['stages']==2 and r['ctas']==(3 if dt=='float64' else 4)]
    print('  default-like:', [(r['ms'], r['gbs']) for r in d])
PY
