# GPU iteration: parity tests, bench line, one ncu --set full capture
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --cpu-budget 0.5 > /dev/null 2> gpurun_out/ncu_$TAG.err
echo "ncu rc=$?"
fi
