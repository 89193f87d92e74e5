# A/B: x gathers with L1::no_allocate (na) / L1::evict_last (el) vs default ld.global.nc
mkdir -p gpurun_out
O=gpurun_out/l1hint; mkdir -p $O
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1; }
for r in 1 2; do
  for cfg in C5 C2 C3 "C5 --fp32"; do
    tag=$(echo $cfg | tr -d ' -')
    for lib in default na el; do
      if [ $lib = default ]; then unset CSRK_LIB; else export CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
      timeout 600 python bench.py --config $cfg --cpu-budget 0.2 > $O/${tag}_${lib}_$r.json 2> $O/${tag}_${lib}_$r.err
      summ $O/${tag}_${lib}_$r.json
    done
  done
done
