mkdir -p gpurun_out
TAG=${1:-ah}
timeout 900 python -m pytest tests -x -q -m gpu -k "schedules or sliced or tile_plans or pinned or auto_plan or c4_full or golden or parity" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
SWEEP_VARIANTS=serial SWEEP_GATHER=0,3 SWEEP_CTAS=0,2,3 SWEEP_TILES=1536,2048 SWEEP_STAGES=2,3 SWEEP_DTYPES=float64 timeout 900 python tools/plan_sweep.py C5 C2 > gpurun_out/sweep_$TAG.txt 2> gpurun_out/sweep_$TAG.err
python tools/sweep_table.py gpurun_out/sweep_$TAG.txt
