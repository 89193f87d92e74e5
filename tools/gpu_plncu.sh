mkdir -p gpurun_out
for cfg in "20000 serial 0" "20000 strided 4"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 2 -c 1 \
    -o gpurun_out/pl_$1_$2_$3 -f python tools/pl_one.py $1 $2 $3 > gpurun_out/pl_ncu_$1_$2_$3.log 2>&1
  python tools/ncu_summary.py gpurun_out/pl_$1_$2_$3.ncu-rep > gpurun_out/pl_ncu_$1_$2_$3.txt 2>&1
  echo "== $cfg"; head -34 gpurun_out/pl_ncu_$1_$2_$3.txt | grep -v "launch__\|  [a-z_]* *[0-9]*$"; grep plan gpurun_out/pl_ncu_$1_$2_$3.log
done
