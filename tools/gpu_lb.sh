mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or schedules or tile_plans or auto_plan or long_rows" > gpurun_out/pytest_lb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lb.log
tail -2 gpurun_out/pytest_lb.log
SWEEP_NX=2,4,8 SWEEP_VARIANTS=serial,strided SWEEP_GATHER=2 SWEEP_CTAS=0 SWEEP_TILES=0 SWEEP_STAGES=0 SWEEP_DTYPES=float64,float32 timeout 600 python tools/plan_sweep.py C3 C5 C2 > gpurun_out/sweep_lb2.txt 2>/dev/null
python tools/sweep_table.py gpurun_out/sweep_lb2.txt
timeout 600 python bench.py --config C3 --steps 100 --warmup 5 --cpu-budget 1 > gpurun_out/bench_C3_lb.json 2>/dev/null; cat gpurun_out/bench_C3_lb.json
