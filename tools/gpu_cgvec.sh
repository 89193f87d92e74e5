# A/B of the fp32 CG BLAS-1 kernels: float4 + fp32 arithmetic (default build)
# against the scalar fp64-arithmetic kernels (SRC=cg build_variant cgscalar)
mkdir -p gpurun_out
O=gpurun_out/cgvec; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cg.py tests/test_dist.py -x -q -m gpu > $O/pytest_cg.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_cg.log
for r in 1 2; do
  for lib in default cgscalar; do
    if [ $lib = default ]; then unset CSRK_LIB; else export CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
    timeout 600 python bench.py --config C4 --fp32 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f32_${lib}_$r.json 2> $O/C4f32_${lib}_$r.err; echo "C4f32 $lib $r rc=$?"
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['config']['ms_per_iteration'], d['roofline']['frac'], d['clocks'])" $O/C4f32_${lib}_$r.json
  done
done
unset CSRK_LIB
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f64.json 2> $O/C4f64.err; echo "C4f64 rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['config']['ms_per_iteration'], d['roofline']['frac'], d['clocks'])" $O/C4f64.json
