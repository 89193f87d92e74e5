"""Kernel-driven PCIe copies (SM loads / stores on mapped pinned memory) vs
copy-engine copies, alone and concurrently.  python tools/pcie_kernel_probe.py"""
import time

import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <cuda_runtime.h>
#include <torch/extension.h>
__global__ void copy16(const int4* __restrict__ s, int4* __restrict__ d, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    int4 a = s[i], b = s[i + st], c = s[i + 2 * st], e = s[i + 3 * st];
    d[i] = a; d[i + st] = b; d[i + 2 * st] = c; d[i + 3 * st] = e;
  }
  for (; i < n; i += st) d[i] = s[i];
}
void kcopy(long src, long dst, long bytes, long stream, int blocks) {
  copy16<<<blocks, 512, 0, (cudaStream_t)stream>>>((const int4*)src, (int4*)dst, bytes / 16);
}
void* dev_alias(long p) { void* d = nullptr; cudaHostGetDevicePointer(&d, (void*)p, 0); return d; }
long alias(long p) { return (long)dev_alias(p); }
"""
mod = load_inline("pcie_kprobe", cpp_sources="void kcopy(long,long,long,long,int); long alias(long);",
                  cuda_sources=src, functions=["kcopy", "alias"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"], verbose=False)

n = 1 << 24
xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.empty(n, dtype=torch.float64, device="cuda")
xa, ya = mod.alias(xh.data_ptr()), mod.alias(yh.data_ptr())
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for blocks in (148, 296, 592):
    k_h2d = lambda: mod.kcopy(xa, xd.data_ptr(), B, s1.cuda_stream, blocks)
    k_d2h = lambda: mod.kcopy(yd.data_ptr(), ya, B, s2.cuda_stream, blocks)
    print(f"blocks {blocks}: kernel H2D {t(k_h2d):.3f} ms  kernel D2H {t(k_d2h):.3f} ms")

    def ce_h2d_k_d2h():
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
        k_d2h()

    def k_h2d_ce_d2h():
        k_h2d()
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)

    def k_both():
        k_h2d()
        k_d2h()
    print(f"  CE H2D + kernel D2H {t(ce_h2d_k_d2h):.3f} ms; kernel H2D + CE D2H "
          f"{t(k_h2d_ce_d2h):.3f} ms; kernel both {t(k_both):.3f} ms")


def both():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)


print(f"CE both {t(both):.3f} ms; CE H2D {t(lambda: xd.copy_(xh, non_blocking=True)):.3f} ms")
