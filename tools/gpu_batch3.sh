mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_b3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b3.log
tail -40 gpurun_out/pytest_b3.log
timeout 600 python bench.py --steps 100 --warmup 10 --cpu-budget 3 > gpurun_out/bench_b3.json 2> gpurun_out/bench_b3.err; cat gpurun_out/bench_b3.json
timeout 900 python bench.py --config C4 --loop cg --steps 3 --warmup 1 > gpurun_out/bench_C4_cg.json 2> gpurun_out/bench_C4_cg.err; cat gpurun_out/bench_C4_cg.json; tail -3 gpurun_out/bench_C4_cg.err
timeout 900 python bench.py --config C4 --loop cg --fp32 --steps 3 --warmup 1 > gpurun_out/bench_C4_cg32.json 2> gpurun_out/bench_C4_cg32.err; cat gpurun_out/bench_C4_cg32.json; tail -3 gpurun_out/bench_C4_cg32.err
timeout 1200 python tools/plan_sweep.py C2 C3 C5 > gpurun_out/plan_sweep.log 2>&1; tail -5 gpurun_out/plan_sweep.log
