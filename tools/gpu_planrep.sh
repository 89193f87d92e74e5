mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_abi.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/planrep_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/planrep_pytest.log
timeout 600 python bench.py --config C2 --fp32 --cpu-budget 0.2 > gpurun_out/planrep_C2f32.json 2>/dev/null; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/planrep_C2f32.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['config']['plan'])"
