# new auto for irregular rows without long rows (1536 x 2 x 3): C5 and power-law capped at 128 / 64
# against the round-1 irregular plan (2048 x 2 x 2); bench lines; power-law with long rows unchanged; GPU suite
mkdir -p gpurun_out
O=gpurun_out/c5auto; mkdir -p $O
for spec in "C5 2048 2 2" "C5 2048 2 2 --fp32" "PL128 2048 2 2" "PL64 2048 2 2" "PL128 2048 2 2 --fp32"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee $O/plan_confirm.jsonl
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['config']['plan'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for c in C5 "C5 --fp32"; do tag=$(echo $c | tr -d ' -'); timeout 600 python bench.py --config $c --cpu-budget 0.2 > $O/$tag.json 2> $O/$tag.err; summ $O/$tag.json; done
timeout 600 python tools/powerlaw_probe.py 2000000 20000 2>&1 | tail -6 | tee $O/powerlaw20k.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
