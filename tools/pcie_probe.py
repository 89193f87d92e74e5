"""PCIe probe for the host pipeline: big vs chunked copies, with and without
concurrent SpMV kernels (C2 sizes).  python tools/pcie_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

n = 1 << 24
xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.empty(n, dtype=torch.float64, device="cuda")
big = torch.empty(1 << 28, dtype=torch.float64, device="cuda")  # 2 GB HBM churn
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def chunked(k, with_kernel=False, ordered=False):
    def fn():
        step = n // k
        evs = []
        with torch.cuda.stream(s1):
            for c in range(k):
                xd[c * step:(c + 1) * step].copy_(xh[c * step:(c + 1) * step], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        for c in range(k):
            if with_kernel:
                with torch.cuda.stream(s3):
                    if ordered:
                        s3.wait_event(evs[c])
                    big[: 1 << 24].add_(1.0)  # ~0.4 GB of HBM traffic
                    e = torch.cuda.Event()
                    e.record(s3)
                if ordered:
                    s2.wait_event(e)
            with torch.cuda.stream(s2):
                yh[c * step:(c + 1) * step].copy_(yd[c * step:(c + 1) * step], non_blocking=True)
    return fn


sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def alternating(k, nstreams=2):
    """kernel c and D2H c in order on comp stream c % nstreams (no
    cross-stream wait in front of a copy, only in front of kernels)."""
    comps = [sa, sb, s3][:nstreams]

    def fn():
        step = n // k
        evs = []
        with torch.cuda.stream(s1):
            for c in range(k):
                xd[c * step:(c + 1) * step].copy_(xh[c * step:(c + 1) * step], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        for c in range(k):
            st = comps[c % nstreams]
            st.wait_event(evs[c])
            with torch.cuda.stream(st):
                big[: 1 << 24].add_(1.0)
                yh[c * step:(c + 1) * step].copy_(yd[c * step:(c + 1) * step], non_blocking=True)
    return fn


def host_ordered(k):
    """D2H c enqueued by the host once kernel c has finished."""
    def fn():
        step = n // k
        evs = []
        with torch.cuda.stream(s1):
            for c in range(k):
                xd[c * step:(c + 1) * step].copy_(xh[c * step:(c + 1) * step], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        kev = []
        for c in range(k):
            s3.wait_event(evs[c])
            with torch.cuda.stream(s3):
                big[: 1 << 24].add_(1.0)
                e = torch.cuda.Event()
                e.record(s3)
                kev.append(e)
        for c in range(k):
            kev[c].synchronize()
            with torch.cuda.stream(s2):
                yh[c * step:(c + 1) * step].copy_(yd[c * step:(c + 1) * step], non_blocking=True)
    return fn


print(f"H2D big        {t(lambda: xd.copy_(xh, non_blocking=True)):.3f} ms")
print(f"D2H big        {t(lambda: yh.copy_(yd, non_blocking=True)):.3f} ms")


def both():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)


print(f"both big       {t(both):.3f} ms")
for k in (8, 16):
    print(f"alternating2 {k:3d}             {t(alternating(k)):.3f} ms")
    print(f"alternating3 {k:3d}             {t(alternating(k, 3)):.3f} ms")
    print(f"host-ordered {k:3d}             {t(host_ordered(k)):.3f} ms")
for k in (4, 8, 16, 64):
    print(f"both chunked {k:3d}             {t(chunked(k)):.3f} ms")
    print(f"both chunked {k:3d} +kernel     {t(chunked(k, True)):.3f} ms")
    print(f"both chunked {k:3d} +kernel ord {t(chunked(k, True, True)):.3f} ms")
