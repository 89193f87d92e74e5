mkdir -p gpurun_out
SWEEP_DTYPES=float64 SWEEP_VARIANTS=strided SWEEP_NX=8,16,32 SWEEP_GATHER=0,1 SWEEP_CTAS=0 SWEEP_TILES=0 SWEEP_STAGES=0 \
  timeout 900 python tools/plan_sweep.py C5 PL64 C1 > gpurun_out/sg_sweep.txt 2> gpurun_out/sg_sweep.err
python tools/sweep_table.py gpurun_out/sg_sweep.txt
