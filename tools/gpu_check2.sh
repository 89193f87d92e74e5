mkdir -p gpurun_out
TAG=${1:-r01e}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for C in C3 C2 C5; do timeout 600 python bench.py --config $C --steps 100 --warmup 5 --cpu-budget 2 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; done
