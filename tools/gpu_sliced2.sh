mkdir -p gpurun_out
TAG=${1:-sl}
SWEEP_VARIANTS=serial SWEEP_GATHER=0 SWEEP_CTAS=0,3 SWEEP_LAYOUT=0,1 SWEEP_TILES=1536,2048 SWEEP_STAGES=2 SWEEP_DTYPES=float64 timeout 900 python tools/plan_sweep.py C5 C2 > gpurun_out/sweep_$TAG.txt 2> gpurun_out/sweep_$TAG.err
python tools/sweep_table.py gpurun_out/sweep_$TAG.txt
