mkdir -p gpurun_out
for cut in groups rows; do
CSRK_CUT=$cut SWEEP_VARIANTS= SWEEP_GATHER=2 SWEEP_CTAS=0 SWEEP_TILES=1536,2048,2560 SWEEP_STAGES=2 SWEEP_DTYPES=float64,float32 timeout 900 python tools/plan_sweep.py C2 C3 C5 > gpurun_out/sweep_cut_$cut.txt 2>gpurun_out/sweep_cut_$cut.err
echo "== cut $cut"; python tools/sweep_table.py gpurun_out/sweep_cut_$cut.txt
done
