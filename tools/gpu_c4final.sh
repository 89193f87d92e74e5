mkdir -p gpurun_out
O=gpurun_out/c4final; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cg.py tests/test_dist.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['config']['ms_per_iteration'], d['value'], d['roofline']['frac'], d['gpu_launches'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for r in 1 2; do
  timeout 600 python bench.py --config C4 --fp32 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f32_$r.json 2> $O/C4f32_$r.err; summ $O/C4f32_$r.json
  CSRK_FUSED_DOT_F32=1 timeout 600 python bench.py --config C4 --fp32 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f32_fused_$r.json 2> $O/C4f32_fused_$r.err; summ $O/C4f32_fused_$r.json
done
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --cpu-budget 0.2 > $O/C4f64.json 2> $O/C4f64.err; summ $O/C4f64.json
