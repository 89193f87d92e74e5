# Full evidence pass on one B200: tests, smoke, every bench line, the reference
# arm, the torchrun paths, the launch list of the default bench command and
# ncu --set full captures of the dominant kernel per config.
#   bash tools/gpu_evidence.sh r02fin
mkdir -p gpurun_out
TAG=${1:-r02fin}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for cfg in C1 C3 C5; do
  timeout 600 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "bench $cfg rc=$?"
done
for cfg in C1 C2 C3 C5; do
  timeout 600 python bench.py --config $cfg --fp32 > $O/bench_${cfg}f32.json 2> $O/bench_${cfg}f32.err; echo "bench $cfg f32 rc=$?"
done
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench C4 rc=$?"
timeout 900 python bench.py --config C4 --fp32 --steps 5 --warmup 3 > $O/bench_C4f32.json 2> $O/bench_C4f32.err; echo "bench C4 f32 rc=$?"
for mg in torch native; do
  CSRK_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --mg $mg > $O/bench_dist1_$mg.json 2> $O/bench_dist1_$mg.err; echo "dist1 $mg rc=$?"
done
timeout 1500 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
for cfg in ${REF_CFGS-C1 C3 C5}; do
  timeout 900 python bench.py --impl reference --config $cfg > $O/bench_reference_$cfg.json 2> $O/bench_reference_$cfg.err; echo "ref $cfg rc=$?"
done
# launch list of the default bench command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csrk_stream|long_rows" -c 60 --csv --log-file $O/launches_C2_bench.csv \
  python bench.py --steps 20 --warmup 5 --cpu-budget 0.5 > /dev/null 2>&1; echo "ncu launches rc=$?"
for c in "C2" "C2 --fp32" "C3" "C5" "C1"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
    -o $O/${tag}_full python bench.py --config $c --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1
  echo "ncu $c rc=$?"
  # summaries on the box (gpurun brings back at most 64 MiB): key metrics,
  # stall reasons, source-level hot spots; the report itself only for C2 / C5
  python tools/ncu_summary.py $O/${tag}_full.ncu-rep > $O/${tag}_stream_ncu_full.txt 2>&1
  ncu -i $O/${tag}_full.ncu-rep --page raw --csv > $O/${tag}_raw.csv 2>/dev/null
  if [ "$tag" != "C2" ] && [ "$tag" != "C5" ]; then rm -f $O/${tag}_full.ncu-rep; fi
done
for f in $O/bench_*.json; do echo "== $f"; head -c 400 $f; echo; done
