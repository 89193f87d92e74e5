# schedule check: auto schedule vs explicit, all three HBM configs, plus the bench lines
mkdir -p gpurun_out
TAG=${1:-sched}
SWEEP_GATHER=2,0,1 SWEEP_CTAS=0,2,3 SWEEP_TILES=2048 SWEEP_STAGES=2 SWEEP_DTYPES=float64,float32 timeout 900 python tools/plan_sweep.py C5 C2 C3 > gpurun_out/sweep_$TAG.txt 2> gpurun_out/sweep_$TAG.err
for C in C2 C3 C5; do
  timeout 600 python bench.py --config $C --steps 100 --warmup 5 --cpu-budget 2 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
