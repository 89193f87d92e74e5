mkdir -p gpurun_out
out=gpurun_out/san_long.txt; : > $out
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in "1000 serial 0" "1000 strided 4" "64 serial 0"; do
    set -- $cfg
    PL_N=60000 timeout 900 compute-sanitizer --tool $tool --print-limit 3 python tools/pl_one.py $1 $2 $3 1 > gpurun_out/san_tmp.log 2>&1
    echo "$tool max_len=$1 $2 nx=$3 rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_tmp.log | tr '\n' ' ')" | tee -a $out
  done
done
