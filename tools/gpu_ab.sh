# mapping A/B + held-out table, and the x-isolated hit-rate probe under ncu
mkdir -p gpurun_out
timeout 1500 python tools/mapping_ab.py ${AB_CONFIGS:-C1 C2 C3 C5} > gpurun_out/mapping_ab.log 2> gpurun_out/mapping_ab.err; echo "ab rc=$?"
tail -3 gpurun_out/mapping_ab.err
M=$(python tools/x_l2_probe.py --metrics)
timeout 900 ncu --clock-control none -k regex:"gather_probe|csrk_stream" --metrics $M --csv --log-file gpurun_out/x_l2.csv python tools/x_l2_probe.py C1 C2 C3 C5 > gpurun_out/x_l2.out 2> gpurun_out/x_l2.err; echo "ncu rc=$?"
python tools/x_l2_probe.py --summarise gpurun_out/x_l2.csv > gpurun_out/x_l2_summary.jsonl; cat gpurun_out/x_l2_summary.jsonl
timeout 600 python tools/x_l2_probe.py C1 C2 C3 C5 > gpurun_out/x_l2_times.jsonl 2>/dev/null; cat gpurun_out/x_l2_times.jsonl
