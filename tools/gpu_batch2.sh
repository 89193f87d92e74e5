mkdir -p gpurun_out
for c in C3 C5; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 --cpu-budget 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --steps 100 --warmup 10 --cpu-budget 2 > gpurun_out/bench_C2b.json 2> gpurun_out/bench_C2b.err
cat gpurun_out/bench_C3.json gpurun_out/bench_C5.json gpurun_out/bench_C2b.json
timeout 3000 python tools/fit_b200.py gpurun_out/fit_b200_raw.json > gpurun_out/fit_b200.log 2>&1
tail -12 gpurun_out/fit_b200.log
