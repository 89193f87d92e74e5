mkdir -p gpurun_out
SWEEP_FLUSH=1 SWEEP_TILES=768,1024,1536,2048 SWEEP_STAGES=1,2 SWEEP_CTAS=3,6,8,12 SWEEP_DTYPES=float64 SWEEP_GATHER=0 \
  timeout 900 python tools/plan_sweep.py C1 > gpurun_out/c1b.jsonl 2> gpurun_out/c1b.err; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/c1b.jsonl') if l.startswith('{')]
for r in sorted(rows, key=lambda r: r['ms'])[:12]: print(r['tile_cost'], r['stages'], r['ctas'], r['ms'], r['gbs'], r['bitwise_equal'])
print('default', [ (r['ms'],r['gbs']) for r in rows if r['tile_cost']==2048 and r['stages']==2 and r['ctas']==3])
PY
