mkdir -p gpurun_out
cp profiles/r01_fit_b200_raw_v2.json gpurun_out/fit_b200_raw4.json
timeout 1500 python tools/fit_b200.py gpurun_out/fit_b200_raw4.json stencil3d27_l irreg_l79 > gpurun_out/fit_b200_4.log 2>&1
tail -3 gpurun_out/fit_b200_4.log
