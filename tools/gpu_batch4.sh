mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
tail -15 gpurun_out/pytest_full.log
SWEEP_STAGES=2 timeout 1200 python tools/plan_sweep.py C2 C3 C5 > gpurun_out/plan_sweep2.log 2>&1; cp gpurun_out/plan_sweep.json gpurun_out/plan_sweep2.json
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-budget 3 > gpurun_out/bench_b4.json 2> gpurun_out/bench_b4.err; cat gpurun_out/bench_b4.json
