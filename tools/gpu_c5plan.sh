# C5 (irregular, no long rows): candidate plans against the auto plan (2048 x 2 stages x 2 CTAs), interleaved
mkdir -p gpurun_out
for spec in "C5 1536 2 3" "C5 1280 2 3" "C5 1536 2 3 --fp32" "C5 1792 2 3" "C5 2048 2 2 --fp32" "C5 1536 2 4 --fp32"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee gpurun_out/c5_plan_confirm.jsonl
