mkdir -p gpurun_out
for L in 0 1; do
LAYOUT=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:csrk_ -s 3 -c 1 \
  -o gpurun_out/prof_C5_L$L python tools/ncu_plan.py C5 2048 2 0 serial > /dev/null 2>&1
echo "ncu L$L rc=$?"
done
