mkdir -p gpurun_out
O=gpurun_out/c1rot; mkdir -p $O
for c in "C1" "C1 --fp32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --config $c --cpu-budget 0.5 > $O/$tag.json 2> $O/$tag.err; echo "$tag rc=$?"
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity']['ok'], d['single_launch_l2_flushed'], d['config']['l2'], d['clocks'])" $O/$tag.json
done
