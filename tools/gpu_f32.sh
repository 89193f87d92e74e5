mkdir -p gpurun_out
SWEEP_DTYPES=float32 SWEEP_VARIANTS=serial SWEEP_GATHER=0 SWEEP_CTAS=3,4,5,6 SWEEP_TILES=2048,2560,3072,4096 SWEEP_STAGES=2,3 \
  timeout 900 python tools/plan_sweep.py C2 > gpurun_out/f32_sweep.txt 2> gpurun_out/f32_sweep.err
python tools/sweep_table.py gpurun_out/f32_sweep.txt
