"""One power-law matrix, a few SpMVs of one order (ncu target):
    python tools/pl_one.py MAX_LEN VARIANT NX [REPS]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from powerlaw_probe import build_powerlaw, ck  # noqa: E402

max_len, variant, nx = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
a, m, st, p = build_powerlaw(int(os.environ.get("PL_N", 2_000_000)), max_len)
x = torch.rand(a.n_rows, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    ck.spmv_device(m, x, y, dims=ck.BlockDims(max(nx, 1), 1, 1), variant=variant)
torch.cuda.synchronize()
print("plan", m.device().plan())
