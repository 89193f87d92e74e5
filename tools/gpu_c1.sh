mkdir -p gpurun_out
SWEEP_FLUSH=1 SWEEP_DTYPES=float64 SWEEP_VARIANTS=serial SWEEP_GATHER=0,1 SWEEP_CTAS=2,3,4 SWEEP_TILES=1024,1536,2048,3072,4096 SWEEP_STAGES=2,3 \
  timeout 900 python tools/plan_sweep.py C1 > gpurun_out/c1_sweep.txt 2> gpurun_out/c1_sweep.err
python tools/sweep_table.py gpurun_out/c1_sweep.txt
