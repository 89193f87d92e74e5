# C5 with the final plan: bench lines (f64, f32) and one ncu --set full capture
mkdir -p gpurun_out/c5final
O=gpurun_out/c5final
for c in "C5" "C5 --fp32"; do tag=$(echo $c | tr -d ' -'); timeout 600 python bench.py --config $c > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$tag rc=$?"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csrk_stream -s 3 -c 1 -o $O/C5_full python bench.py --config C5 --steps 1 --warmup 3 --cpu-budget 0.2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/C5_full.ncu-rep > $O/C5_stream_ncu_full.txt 2>&1
ncu -i $O/C5_full.ncu-rep --page raw --csv > $O/C5_raw.csv 2>/dev/null
head -20 $O/C5_stream_ncu_full.txt
