mkdir -p gpurun_out
for cfg in "20000 serial 0" "20000 strided 4"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csrk_stream|long_rows_kernel" -s 4 -c 2 \
    -o gpurun_out/plf_$1_$2_$3 -f python tools/pl_one.py $1 $2 $3 > gpurun_out/plf_ncu_$1_$2_$3.log 2>&1
  ncu -i gpurun_out/plf_$1_$2_$3.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/plf_$1_$2_$3.csv 2>&1
  echo "== $cfg"; cut -c1-20,1-0 gpurun_out/plf_$1_$2_$3.csv | head -0; python - "$1_$2_$3" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/plf_{sys.argv[1]}.csv")))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d.get("Kernel Name", "")[:60], {k: d[k] for k in h if "__" in k})
PY
done
