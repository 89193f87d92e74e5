# per-kernel times of the C4 CG iteration (fp32 and fp64) under ncu (serialised, cold)
mkdir -p gpurun_out
for p in "--fp32" ""; do
  tag=C4${p#--}
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base \
    -k regex:"csrk_stream|cg_update|cg_direction|set_rr|dot_partial" -c 24 --csv --log-file gpurun_out/${tag}_split.csv \
    python bench.py --config C4 $p --steps 1 --warmup 3 --iters 4 --cpu-budget 0.2 > /dev/null 2>&1; echo "$tag rc=$?"
  python - gpurun_out/${tag}_split.csv <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); k = d['Kernel Name'].split('(')[0].split('<')[0]
        agg[k][d['Metric Name']].append(float(d['Metric Value'].replace(',', '')))
for k, m in agg.items():
    t = sorted(m['gpu__time_duration.sum']); med = t[len(t)//2]
    rb = sorted(m['dram__bytes_read.sum'])[len(t)//2]; wb = sorted(m['dram__bytes_write.sum'])[len(t)//2]
    print(f"{k:28s} n={len(t):3d} median {med/1e3:8.1f} us  dram {(rb+wb)/1e9:6.3f} GB  -> {(rb+wb)/med:7.1f} GB/s")
PY
done
