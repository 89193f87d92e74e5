# C5: deeper rings of smaller tiles at the same shared-memory budget
mkdir -p gpurun_out
SWEEP_DTYPES=float64 SWEEP_VARIANTS=serial SWEEP_GATHER=0 SWEEP_CTAS=2,3,4 SWEEP_TILES=768,1024,1280 SWEEP_STAGES=2,3,4,5 \
  timeout 1200 python tools/plan_sweep.py C5 > gpurun_out/c5_deep_sweep.jsonl 2> gpurun_out/c5_deep_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/c5_deep_sweep.jsonl') if l.strip().startswith('{')]
for r in sorted(rows, key=lambda r: r.get('ms', 9)):
    print(r.get('ctas'), r.get('tile_cost'), r.get('stages'), r.get('ms'), r.get('bitwise_equal'))
PY
