# row stride between sub-warps (STRIDED order): parity at every stride, then
# A/B auto (C3: stride 4) vs CSRK_ROW_STRIDE=1 (round-2 mapping) interleaved
mkdir -p gpurun_out
O=gpurun_out/rowstride; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_row_stride.py tests/test_gpu_parity.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for r in 1 2 3; do
  for cfg in C3 "C3 --fp32"; do
    tag=$(echo $cfg | tr -d ' -')
    for st in auto 1; do
      if [ $st = auto ]; then unset CSRK_ROW_STRIDE; else export CSRK_ROW_STRIDE=$st; fi
      timeout 600 python bench.py --config $cfg --cpu-budget 0.2 > $O/${tag}_s${st}_$r.json 2> $O/${tag}_s${st}_$r.err
      summ $O/${tag}_s${st}_$r.json
    done
  done
done
unset CSRK_ROW_STRIDE
timeout 900 ncu --set full --clock-control none -k regex:csrk_stream -s 3 -c 1 -o $O/C3_full python bench.py --config C3 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/C3_full.ncu-rep > $O/C3_stream_ncu_full.txt 2>&1; head -20 $O/C3_stream_ncu_full.txt
ncu -i $O/C3_full.ncu-rep --page raw --csv > $O/C3_raw.csv 2>/dev/null; rm -f $O/C3_full.ncu-rep
