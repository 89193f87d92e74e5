mkdir -p gpurun_out
for e in "X=1" "CSRK_LONG_SERIAL=1"; do
echo "== $e"
env $e SWEEP_DTYPES=float64 SWEEP_VARIANTS=strided SWEEP_NX=4,8 SWEEP_GATHER=2 SWEEP_CTAS=0 SWEEP_TILES=1702,2048 SWEEP_STAGES=2 \
  timeout 900 python tools/plan_sweep.py PL20000 2>/dev/null > gpurun_out/nx8.txt
python tools/sweep_table.py gpurun_out/nx8.txt
done
