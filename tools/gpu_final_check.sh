# final check of the tree: GPU suite (incl. the PDL chain tests), smoke, default bench line
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline'], d['e2e'], d['parity']['ok'], d['clocks'], d['gpu_launches'])" $O/bench_default.json
