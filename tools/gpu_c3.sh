mkdir -p gpurun_out
SWEEP_DTYPES=float64 SWEEP_VARIANTS=serial,strided SWEEP_NX=2,4,8 SWEEP_GATHER=0,1,2 SWEEP_CTAS=0,2,3,4 SWEEP_TILES=0 SWEEP_STAGES=0 \
  timeout 900 python tools/plan_sweep.py C3 C2 > gpurun_out/c3_sweep.txt 2> gpurun_out/c3_sweep.err
python tools/sweep_table.py gpurun_out/c3_sweep.txt
