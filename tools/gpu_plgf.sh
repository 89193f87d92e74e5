mkdir -p gpurun_out
for spec in "PL128 1536 2 2" "PL64 1536 2 2" "PL128 2048 2 2" "PL64 2048 2 2" "PL128 1536 2 3 --fp32"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee gpurun_out/plgf.jsonl
