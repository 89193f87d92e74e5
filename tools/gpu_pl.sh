mkdir -p gpurun_out
SWEEP_DTYPES=float64 SWEEP_VARIANTS=serial SWEEP_NX=8 SWEEP_GATHER=0,1 SWEEP_CTAS=1,2,3,4 SWEEP_TILES=1024,2048,4096 SWEEP_STAGES=2 \
  timeout 900 python tools/plan_sweep.py PL64 PL20000 > gpurun_out/pl_sweep.txt 2> gpurun_out/pl_sweep.err
python tools/sweep_table.py gpurun_out/plan_sweep.json > gpurun_out/pl_sweep_table.txt 2>&1 || true
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csrk|long" --csv \
  --log-file gpurun_out/pl_launches.csv python tools/powerlaw_probe.py 2000000 20000 > gpurun_out/pl_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open("gpurun_out/pl_launches.csv") if l.startswith('"')))
agg = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        agg[r["Kernel Name"][:90]].append(float(r["Metric Value"]))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    v.sort(); print(f"{len(v):5d} med {v[len(v)//2]/1e3 if max(v)>1e4 else v[len(v)//2]:10.1f}  {k}")
PY
