# Full GPU evidence pass: parity tests, smoke, both bench arms, per-config
# bench lines, the ncu launch list of the bench command (timed kernel only)
# and one --set full capture of the streaming kernel per config.
# usage: bash tools/gpu_round.sh TAG [CONFIGS...]
mkdir -p gpurun_out
TAG=${1:-r01}
shift
CONFIGS=${@:-C2 C5}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
cat gpurun_out/bench_ref_$TAG.json
for C in $CONFIGS; do
  timeout 600 python bench.py --config $C --steps 100 --warmup 5 --cpu-budget 3 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
done
timeout 600 python bench.py --fp32 --steps 100 --warmup 5 --cpu-budget 1 > gpurun_out/bench_C2f32_$TAG.json 2> gpurun_out/bench_C2f32_$TAG.err
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 > gpurun_out/bench_C4_$TAG.json 2> gpurun_out/bench_C4_$TAG.err
timeout 900 python bench.py --config C4 --fp32 --steps 2 --warmup 3 > gpurun_out/bench_C4f32_$TAG.json 2> gpurun_out/bench_C4f32_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:csrk_stream -c 60 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --cpu-budget 0.5 > gpurun_out/launches_$TAG.out 2>&1
echo "launches rc=$?"
for C in $CONFIGS; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
  -o gpurun_out/prof_${C}_$TAG python bench.py --config $C --steps 1 --warmup 3 --cpu-budget 0.5 > /dev/null 2> gpurun_out/ncu_${C}_$TAG.err
echo "ncu $C rc=$?"
done
ls gpurun_out/ | grep $TAG
