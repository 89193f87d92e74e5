mkdir -p gpurun_out
for c in "C1" "C1 --fp32" "C5 --fp32"; do
  timeout 600 python tools/c1_graph_ab.py $c 64 5 2>> gpurun_out/c1_graph_ab.err; echo "$c rc=$?"
done | tee gpurun_out/c1_graph_ab.jsonl
