"""Iterative callers of the CSR-k SpMV on the device.

BASELINE config C4 is "100 repeated SpMVs as a CG inner loop".  Two loops
run entirely on the GPU through the C-ABI (csrc/cg.cu):

  cg(m, b, ...)           conjugate gradients for SPD A (e.g. the Laplacians)
  power_iterations(m, x)  x <- A x / max|A x|, the repeated-SpMV loop of
                          SURVEY.md §8(d)

Both take torch CUDA tensors, launch on one stream without host
synchronisation, and can be captured once into a CUDA graph
(:class:`GraphedLoop`) and replayed -- the B200 replacement for a
host-driven loop.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .kernels import check_device_vector

__all__ = ["cg", "power_iterations", "GraphedLoop", "device_handle"]


def device_handle(m) -> nat.DeviceMatrix:
    """DeviceMatrix of a CsrMatrix / CsrKMatrix / DeviceMatrix."""
    return m if isinstance(m, nat.DeviceMatrix) else m.device()


def _variant(dims, variant):
    if variant == "strided":
        return nat.CSRK_STRIDED, (dims.x if dims is not None else 1)
    if variant != "serial":
        raise ValueError(f"unknown variant {variant!r}")
    return nat.CSRK_SERIAL, 1


def _vt(t):
    import torch

    if t.dtype == torch.float64:
        return nat.CSRK_F64
    if t.dtype == torch.float32:
        return nat.CSRK_F32
    raise ValueError("vectors must be float32 or float64")


def cg(m, b, x=None, iters: int = 100, *, dims=None, variant: str = "serial",
       stream=None, scratch=None, sync: bool = True):
    """Run ``iters`` CG iterations for A x = b on the device; returns
    ``(x, info)`` with info = {"rr", "alpha", "beta", "pAp"} of the last
    iteration when ``sync`` (else info is None and nothing waits)."""
    import torch

    dev = device_handle(m)
    if dev.n_rows != dev.n_cols:
        raise ValueError("CG requires a square matrix")
    vt = _vt(b)
    check_device_vector(b, dev, dev.n_rows, "b")
    if vt == nat.CSRK_F32:
        dev.ensure_f32()
    if x is None:
        x = torch.zeros_like(b)
    r, p, ap = scratch if scratch is not None else (torch.empty_like(b) for _ in range(3))
    for name, t in (("x", x), ("r", r), ("p", p), ("ap", ap)):
        check_device_vector(t, dev, dev.n_rows, name, dtype=b.dtype)
    var, nx = _variant(dims, variant)
    stream = stream or torch.cuda.current_stream(b.device)
    sc = np.zeros(4) if sync else None
    nat.call("csrk_cg", dev.ptr, vt, var, nx, C.c_void_p(b.data_ptr()),
             C.c_void_p(x.data_ptr()), C.c_void_p(r.data_ptr()), C.c_void_p(p.data_ptr()),
             C.c_void_p(ap.data_ptr()), int(iters), nat.f64p(sc) if sync else None,
             C.c_void_p(stream.cuda_stream))
    info = None
    if sync:
        info = {"rr": float(sc[0]), "alpha": float(sc[1]), "beta": float(sc[2]),
                "pAp": float(sc[3])}
    return x, info


def power_iterations(m, x, iters: int = 100, *, dims=None, variant: str = "serial",
                     y=None, stream=None):
    """``iters`` times x <- A x / max|A x| on the device (x updated in place)."""
    import torch

    dev = device_handle(m)
    if dev.n_rows != dev.n_cols:
        raise ValueError("power iterations require a square matrix")
    vt = _vt(x)
    check_device_vector(x, dev, dev.n_cols, "x")
    if vt == nat.CSRK_F32:
        dev.ensure_f32()
    y = torch.empty_like(x) if y is None else y
    check_device_vector(y, dev, dev.n_rows, "y", dtype=x.dtype)
    var, nx = _variant(dims, variant)
    stream = stream or torch.cuda.current_stream(x.device)
    nat.call("csrk_power", dev.ptr, vt, var, nx, C.c_void_p(x.data_ptr()),
             C.c_void_p(y.data_ptr()), int(iters), C.c_void_p(stream.cuda_stream))
    return x


class GraphedLoop:
    """Capture ``fn(stream)`` once into a CUDA graph and replay it."""

    def __init__(self, fn, device=None):
        import torch

        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=device)
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            fn(s)  # warm-up outside capture (plans, attributes)
        torch.cuda.current_stream(device).wait_stream(s)
        torch.cuda.synchronize(device)
        with torch.cuda.graph(self.graph, stream=s):
            fn(s)

    def replay(self):
        self.graph.replay()
