mkdir -p gpurun_out
for W in 8 12 16; do
CSRK_SLICED_WARPS=$W SWEEP_VARIANTS=serial SWEEP_GATHER=0 SWEEP_CTAS=1,2,3 SWEEP_LAYOUT=1 SWEEP_TILES=1536,2048 SWEEP_STAGES=2 SWEEP_DTYPES=float64 timeout 600 python tools/plan_sweep.py C5 C2 > gpurun_out/sweep_slw$W.txt 2> gpurun_out/sweep_slw$W.err
echo "== W=$W"; python tools/sweep_table.py gpurun_out/sweep_slw$W.txt
done
