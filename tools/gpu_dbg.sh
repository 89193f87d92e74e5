mkdir -p gpurun_out
PL_N=200000 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/pl_one.py 1000 strided 4 1 > gpurun_out/dbg_san.log 2>&1; echo "san rc=$?"
grep -v "^=========     " gpurun_out/dbg_san.log | tail -5
bash tools/gpu_pl2.sh
