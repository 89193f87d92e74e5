mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python tools/c1_flush_ab.py C1 20 5 > gpurun_out/c1_flush_ab.jsonl 2> gpurun_out/c1_flush_ab.err; echo "c1 rc=$?"
cat gpurun_out/c1_flush_ab.jsonl
