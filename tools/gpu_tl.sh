mkdir -p gpurun_out
export CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_tl.so
for c in C1 C2 C5; do
timeout 600 python tools/timeline_probe.py $c 3 > gpurun_out/tl_$c.jsonl 2> gpurun_out/tl_$c.err; echo "$c rc=$?"; cat gpurun_out/tl_$c.jsonl
done
