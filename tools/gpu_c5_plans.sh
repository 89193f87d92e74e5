mkdir -p gpurun_out
timeout 300 python tools/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1
for spec in "1536 2 0 serial" "2048 2 0 serial" "1536 2 1 serial"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o gpurun_out/prof_C5_T$1_S$2_G$3_$4 python tools/ncu_plan.py C5 $1 $2 $3 $4 > /dev/null 2>&1
  echo "ncu $spec rc=$?"
done
