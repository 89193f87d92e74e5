# refined auto (3-stage ring at tile 1536 for regular rows only): in-process interleaved A/Bs + GPU tests
mkdir -p gpurun_out
timeout 600 python tools/c4_plan_ab.py 2>/dev/null | tee gpurun_out/c4_plan_ab.jsonl
timeout 600 python tools/c4_plan_ab.py --fp32 2>/dev/null | tee -a gpurun_out/c4_plan_ab.jsonl
for spec in "C3 1685 2 3" "C2 2048 2 3" "C1 2048 2 3" "C3 1685 2 4 --fp32" "C2 2048 2 4 --fp32" "C5 2048 2 2"; do
  timeout 600 python tools/plan_confirm.py $spec 2>/dev/null
done | tee gpurun_out/plan_confirm3.jsonl
for lib in default oldauto; do
  if [ $lib = default ]; then L=""; else L=paper_2203_05096_b200/lib/libcsrk_cuda_$lib.so; fi
  echo "== powerlaw $lib"; CSRK_LIB=$L timeout 600 python tools/powerlaw_probe.py 2000000 20000 2>&1 | tail -6
done 2>&1 | tee gpurun_out/newauto2_powerlaw.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_newauto2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_newauto2.log; tail -2 gpurun_out/pytest_newauto2.log
