"""Sustained (power-capped) throughput of the streaming kernel under two
layouts / schedules: 3000 back-to-back launches each, alternating.
    python tools/sustained.py [C2]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
dev = m.device()
xd = torch.from_numpy(xp).cuda()
yd = torch.empty_like(xd)
byts = spmv_bytes(a.n_rows, a.n_rows, a.nnz, 8)
for rep in range(2):
    for layout in (0, 1):  # cut mode: auto, rows
        dev.set_cut_mode(layout)
        ck.spmv_device(m, xd, yd)
        torch.cuda.synchronize()
        with bench.ClockSampler(0) as clk:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3000):
                ck.spmv_device(m, xd, yd)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3000
        print(f"{cfg} layout {layout}: {byts / ms / 1e6:.0f} GB/s  {clk.summary()}", flush=True)
        time.sleep(2)
