mkdir -p gpurun_out
TAG=${1:-pf}
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or schedules or tile_plans or pinned or auto_plan or sliced or slabs" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
SWEEP_VARIANTS=serial,strided SWEEP_GATHER=2 SWEEP_CTAS=0 SWEEP_TILES=1024,1536,2048 SWEEP_STAGES=2 SWEEP_DTYPES=float64 timeout 900 python tools/plan_sweep.py C5 C2 C3 > gpurun_out/sweep_$TAG.txt 2>/dev/null
python tools/sweep_table.py gpurun_out/sweep_$TAG.txt
