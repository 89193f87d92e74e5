mkdir -p gpurun_out
TAG=${1:-sl}
timeout 900 python -m pytest tests -x -q -m gpu -k "sliced or schedules or tile_plans or pinned or pipeline_shapes or auto_plan or c4_full" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
SWEEP_VARIANTS=serial SWEEP_GATHER=0 SWEEP_CTAS=0,2,3 SWEEP_LAYOUT=0,1 SWEEP_TILES=1536,2048,3072 SWEEP_STAGES=2,3 SWEEP_DTYPES=float64 timeout 900 python tools/plan_sweep.py C5 C2 C3 > gpurun_out/sweep_$TAG.txt 2> gpurun_out/sweep_$TAG.err
python tools/sweep_table.py gpurun_out/sweep_$TAG.txt
