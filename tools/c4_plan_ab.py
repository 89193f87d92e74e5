"""C4's SpMV (512^3 7-point, natural order, uniform 8 / 8 groups, generated
in HBM) under two explicit plans, interleaved in one process: the round-2
auto plan for regular rows (tile 1536, 3 stages) against round 1's (tile
2048, 2 stages), 3 CTAs per SM, fp64 (and fp32 with --fp32, 4 CTAs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_05096_b200 import _native as nat  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def main():
    f32 = "--fp32" in sys.argv
    side = 512
    dev = synthetic.device_stencil((side, side, side), 7).group_uniform(8, 8)
    if f32:
        dev.ensure_f32()
    dt = torch.float32 if f32 else torch.float64
    n = dev.n_rows
    x = torch.rand(n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    ctas = 4 if f32 else 3

    def timed(k=20):
        for _ in range(3):
            dev.spmv_ptr(x.data_ptr(), y.data_ptr(), s, f32=f32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            dev.spmv_ptr(x.data_ptr(), y.data_ptr(), s, f32=f32)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    res = {"1536x3": [], "2048x2": []}
    for _ in range(4):
        for name, (tc, st) in (("1536x3", (1536, 3)), ("2048x2", (2048, 2))):
            dev.set_plan(tc, 0, st)
            dev.set_schedule(2, ctas)
            res[name].append(round(timed(), 4))
    nb = spmv_bytes(n, n, dev.nnz, 4 if f32 else 8)
    print(json.dumps({"config": "C4 SpMV", "f32": f32, "ms": res,
                      "frac": {k: round(nb / (min(v) * 1e-3) / 1e9 / 6464.3, 4)
                               for k, v in res.items()}}), flush=True)


if __name__ == "__main__":
    main()
