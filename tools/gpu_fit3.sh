mkdir -p gpurun_out
rm -f gpurun_out/fit_b200_raw3.json
timeout 3500 python tools/fit_b200.py gpurun_out/fit_b200_raw3.json stencil2d5 stencil3d7 stencil2d9 stencil3d27 irreg_l5 irreg_l11 irreg_l19 irreg_l39 > gpurun_out/fit_b200_3.log 2>&1
tail -12 gpurun_out/fit_b200_3.log
