# compute-sanitizer audit of the round-2 kernel changes on small inputs:
# predicated asm gathers, ring counters, fused CG dot epilogue, x prefetch,
# multi-GPU C-ABI (one GPU), gather probe
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san2_smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$?"
done
timeout 1500 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "tile_plans or schedules or edge or long_rows or cut_modes" > gpurun_out/san2_parity_memcheck.txt 2>&1
echo "parity memcheck rc=$?"
timeout 1500 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_cg.py > gpurun_out/san2_cg_memcheck.txt 2>&1
echo "cg memcheck rc=$?"
timeout 900 $S --tool synccheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_cg.py -k fused > gpurun_out/san2_cg_synccheck.txt 2>&1
echo "cg fused synccheck rc=$?"
timeout 900 $S --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_cg.py -k fused > gpurun_out/san2_cg_racecheck.txt 2>&1
echo "cg fused racecheck rc=$?"
timeout 1500 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_dist.py -k "native" > gpurun_out/san2_mg_memcheck.txt 2>&1
echo "mg memcheck rc=$?"
for f in gpurun_out/san2_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -3; done
