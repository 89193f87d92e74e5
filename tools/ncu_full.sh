# one ncu --set full capture of the streaming kernel on the bench workload
mkdir -p gpurun_out
CFG=${1:-C2}
NAME=${2:-prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 \
  -o gpurun_out/$NAME python bench.py --config $CFG --steps 1 --warmup 3 --cpu-budget 0.5 > gpurun_out/$NAME.out 2> gpurun_out/$NAME.err
echo "ncu rc=$?"
ls -la gpurun_out/
