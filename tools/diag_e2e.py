"""PCIe / pipeline diagnostics for the host-buffer path (C2)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2203_05096_b200 as ck

a, m, xp, params, _ = bench.build_matrix("C2", lambda s: print(s, file=sys.stderr))
n = a.n_rows
x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
h2d = t(lambda: xd.copy_(x_pin, non_blocking=True))
d2h = t(lambda: y_pin.copy_(yd, non_blocking=True))
def both():
    with torch.cuda.stream(s1): xd.copy_(x_pin, non_blocking=True)
    with torch.cuda.stream(s2): y_pin.copy_(yd, non_blocking=True)
bo = t(both)
print(f"H2D 134MB {h2d:.3f} ms ({n*8/h2d/1e6:.1f} GB/s); D2H {d2h:.3f} ms ({n*8/d2h/1e6:.1f} GB/s); concurrent {bo:.3f} ms")
xn, yn = x_pin.numpy(), y_pin.numpy()
xn[:] = xp
e2e = t(lambda: ck.spmv_csr3(m, xn, out=yn), reps=20)
print(f"e2e spmv_csr3 pinned {e2e:.3f} ms")
dev = m.device()
import ctypes
print("plan", dev.plan())
import os
os.environ["CSRK_PIPE_TRACE"] = "1"
ck.spmv_csr3(m, xn, out=yn)
del os.environ["CSRK_PIPE_TRACE"]
