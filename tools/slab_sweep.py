"""Natural-order 7-point 256^3 (the weak-scaling slab) under several group
sizes and tile plans: python tools/slab_sweep.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def med(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


n = 256 ** 3
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for srs, ssrs in ((8, 8), (4, 16), (16, 16), (32, 8), (1, 1)):
    dev = synthetic.device_stencil((256, 256, 256), 7).group_uniform(srs, ssrs)
    byts = spmv_bytes(n, n, dev.nnz, 8)
    for tc in (0, 1536, 2560, 3072):
        dev.set_plan(tc, 0, 0)
        ms = med(lambda: ck.spmv_device(dev, x, y))
        print(f"srs {srs:2d} ssrs {ssrs:2d} tile {tc or 'auto':>5} {byts / ms / 1e6:7.0f} GB/s "
              f"plan {dev.plan()['n_tiles']} tiles aligned {dev.plan()['group_aligned']}",
              flush=True)
    del dev
