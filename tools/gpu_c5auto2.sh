# refined irregular auto: C5 (inline class) -> 1536 x 2 x 3; power-law (wide spread) -> 2048 x 2 x 2
mkdir -p gpurun_out
O=gpurun_out/c5auto2; mkdir -p $O
for spec in "C5 2048 2 2" "C5 2048 2 2 --fp32" "PL128 1536 2 3" "PL64 1536 2 3"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee $O/plan_confirm.jsonl
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['config']['plan'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for c in C5 "C5 --fp32"; do tag=$(echo $c | tr -d ' -'); timeout 600 python bench.py --config $c --cpu-budget 0.2 > $O/$tag.json 2> $O/$tag.err; summ $O/$tag.json; done
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
