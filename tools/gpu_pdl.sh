# A/B: programmatic dependent launch of the streaming kernel (default) vs
# CSRK_PDL=0, interleaved bench lines; then the GPU suite with PDL on
mkdir -p gpurun_out
O=gpurun_out/pdl; mkdir -p $O
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'] if 'parity' in d else '', d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for r in 1 2; do
  for cfg in C2 C1 C3 C5; do
    for pdl in 1 0; do
      CSRK_PDL=$pdl timeout 600 python bench.py --config $cfg --cpu-budget 0.2 > $O/${cfg}_pdl${pdl}_$r.json 2> $O/${cfg}_pdl${pdl}_$r.err
      summ $O/${cfg}_pdl${pdl}_$r.json
    done
  done
done
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
