bash tools/gpu_pf.sh
AB_CONFIGS="C5 C3" timeout 1500 python tools/mapping_ab.py C5 C3 > gpurun_out/mapping_ab2.log 2> gpurun_out/mapping_ab2.err; echo "ab rc=$?"
