# compute-sanitizer audit of the kernels on small inputs
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 $S --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$?"
done
timeout 1500 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "tile_plans or schedules or sliced or edge or long_rows" > gpurun_out/sanitize_parity_memcheck.txt 2>&1
echo "parity memcheck rc=$?"
timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -m gpu tests/test_gpu_construct.py -k "coo or wbo or radix" > gpurun_out/sanitize_construct_memcheck.txt 2>&1
echo "construct memcheck rc=$?"
tail -3 gpurun_out/sanitize_*.txt
