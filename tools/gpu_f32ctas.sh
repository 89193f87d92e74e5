mkdir -p gpurun_out
for spec in "C2 1536 3 3 --fp32" "C3 1536 3 3 --fp32" "C3 1536 2 4 --fp32" "C2 1536 2 4 --fp32"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee gpurun_out/f32ctas.jsonl
