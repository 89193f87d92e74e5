mkdir -p gpurun_out
python tools/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1
for c in C3 C5 C1; do timeout 900 python bench.py --config $c --steps 100 --warmup 10 --cpu-budget 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config C2 --fp32 --steps 100 --warmup 10 --cpu-budget 2 > gpurun_out/bench_C2_f32.json 2> gpurun_out/bench_C2_f32.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:csrk_stream -s 5 -c 20 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 20 --warmup 5 --cpu-budget 0.5 > /dev/null 2>&1
cat gpurun_out/diag_e2e.txt; for f in gpurun_out/bench_C*.json; do echo $f; cat $f; done
