# C4 fp32: fused p.Ap vs separate dot, and the 2x-unrolled direction kernel (variant build)
mkdir -p gpurun_out
O=gpurun_out/c4ab2; mkdir -p $O
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['config']['ms_per_iteration'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for r in 1 2; do
  for mode in default nofuse unroll; do
    unset CSRK_LIB CSRK_NO_FUSED_DOT
    [ $mode = nofuse ] && export CSRK_NO_FUSED_DOT=1
    [ $mode = unroll ] && export CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_unroll.so
    timeout 600 python bench.py --config C4 --fp32 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f32_${mode}_$r.json 2> $O/C4f32_${mode}_$r.err
    summ $O/C4f32_${mode}_$r.json
  done
done
unset CSRK_LIB CSRK_NO_FUSED_DOT
for mode in nofuse unroll; do
  unset CSRK_LIB CSRK_NO_FUSED_DOT
  [ $mode = nofuse ] && export CSRK_NO_FUSED_DOT=1
  [ $mode = unroll ] && export CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_unroll.so
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base \
    -k regex:"csrk_stream|cg_update|cg_direction|set_rr|dot_partial" -c 24 --csv --log-file $O/split_$mode.csv \
    python bench.py --config C4 --fp32 --steps 1 --warmup 3 --iters 4 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu $mode rc=$?"
  python - $O/split_$mode.csv <<'PY'
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
