mkdir -p gpurun_out
rm -f gpurun_out/fit_b200_raw2.json
timeout 3300 python tools/fit_b200.py gpurun_out/fit_b200_raw2.json > gpurun_out/fit_b200_2.log 2>&1
tail -12 gpurun_out/fit_b200_2.log
