"""SpMV entry points over CSR and CSR-k storage, executed on the B200.

Drop-in for the reference's ``csrk.kernels`` (pkg/src/csrk/kernels.py).
Every function keeps the reference's signature, checks and return type, and
runs a hand-written sm_100a kernel from libcsrk_cuda.so:

  reference function (kernels.py)     device kernel (csrc/spmv.cu)       bits
  ---------------------------------   ---------------------------------  ----------------
  spmv_csr_ref        97-114          csrk_stream_kernel, k=1, SERIAL    == reference
  spmv_csr2           185-206         csrk_stream_kernel, k=2, SERIAL    == reference
  spmv_csr3           209-221         csrk_stream_kernel, k=3, SERIAL    == reference
  emulate_gpu_spmv3   231-261         listing3_kernel (+ lane trace)     == reference
  emulate_gpu_spmv35  284-324         listing4_kernel (+ lane trace)     == reference
  spmv_gpu35 (new)                    csrk_stream_kernel, STRIDED(nx)    == emulate_gpu_spmv35

The serial kernels accumulate each row left to right with separately
rounded multiply and add (no FMA), so y is bitwise the reference's
(SURVEY.md §8(c)).  ``workers`` / ``executor`` are accepted for signature
compatibility; the GPU grid replaces the reference's thread pool and, as in
the reference (kernels.py:202), the result does not depend on them.

Device-resident use (x, y already in HBM) goes through :func:`spmv_device`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .format import VALUE_DTYPE, CsrKMatrix, CsrMatrix

__all__ = [
    "MAX_BLOCK_THREADS",
    "BlockDims",
    "EmulationTrace",
    "spmv_csr_ref",
    "spmv_csr2",
    "spmv_csr3",
    "emulate_gpu_spmv3",
    "emulate_gpu_spmv35",
    "spmv_gpu35",
    "spmv_device",
    "check_device_vector",
    "host_row_sums",
    "STRIDED_NX",
]

MAX_BLOCK_THREADS = 1024  # kernels.py:33

# nx values the streaming STRIDED kernel is instantiated for
STRIDED_NX = tuple(range(1, 17)) + (20, 24, 28, 32)


@dataclass(frozen=True)
class BlockDims:
    """CUDA block shape (x, y, z), each >= 1, at most 1024 threads
    (kernels.py:36-52)."""

    x: int
    y: int
    z: int = 1

    def __post_init__(self) -> None:
        for axis in ("x", "y", "z"):
            if getattr(self, axis) < 1:
                raise ValueError(f"block dimension {axis} must be at least 1")
        total = self.x * self.y * self.z
        if total > MAX_BLOCK_THREADS:
            raise ValueError(f"block holds {total} threads, limit is {MAX_BLOCK_THREADS}")


@dataclass(eq=False)
class EmulationTrace:
    """Per-row lane assignment (kernels.py:55-87): block, z / y lane, first
    x lane and x-lane count, reduction-tree depth.  Produced by the CUDA
    listing kernels themselves, one record per row in row order."""

    row: np.ndarray
    block: np.ndarray
    z_lane: np.ndarray
    y_lane: np.ndarray
    x_first: np.ndarray
    x_count: np.ndarray
    reduction_depth: np.ndarray

    @classmethod
    def from_records(cls, records: list) -> "EmulationTrace":
        table = np.array(records, dtype=np.int64).reshape(-1, 7)
        return cls(*(np.ascontiguousarray(table[:, i]) for i in range(7)))

    def __len__(self) -> int:
        return int(self.row.shape[0])

    def validate_partition(self, n_rows: int) -> None:
        """Raise unless every row 0..n_rows-1 appears exactly once."""
        if self.row.shape[0] != n_rows or not np.array_equal(np.sort(self.row),
                                                             np.arange(n_rows)):
            raise ValueError("trace does not assign every row exactly once")


def _check_x(a: CsrMatrix, x) -> np.ndarray:
    x = np.asarray(x, dtype=VALUE_DTYPE)
    if x.ndim != 1 or x.shape[0] != a.n_cols:
        raise ValueError(f"x must have length {a.n_cols}, got {x.shape}")
    return x


def host_row_sums(row_ptr, col_idx, vals, x) -> np.ndarray:
    """Rows summed strictly left to right on the host, numpy: the product
    ``vals[p] * x[col[p]]`` and each ``acc + prod`` rounded separately, as
    the reference's sequential oracle (kernels.py:97-114) does one Python
    float at a time.  Rows are visited longest first so that step j adds
    entry j of a prefix of the rows (one vectorised add per column
    position, total work nnz)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    n = rp.shape[0] - 1
    y = np.zeros(n, dtype=VALUE_DTYPE)
    if n == 0 or rp[-1] == 0:
        return y
    prods = np.asarray(vals, dtype=VALUE_DTYPE) * x[np.asarray(col_idx, dtype=np.int64)]
    lens = np.diff(rp)
    order = np.argsort(-lens, kind="stable")
    starts = rp[:-1][order]
    sl = lens[order]
    acc = np.zeros(n, dtype=VALUE_DTYPE)
    active = n
    for j in range(int(sl[0])):
        while active > 0 and sl[active - 1] <= j:
            active -= 1
        acc[:active] += prods[starts[:active] + j]
    y[order] = acc
    return y


def spmv_csr_ref(a: CsrMatrix, x, *, out=None) -> np.ndarray:
    """Plain CSR y = A x, rows summed left to right (kernels.py:97-114).

    The reference keeps this as its sequential host oracle, and so does this
    package: it runs on the host (numpy, bitwise the
    reference's per-row chain) and is what run_benchmark / the CLI verify
    the device kernels against.  It is not a fallback of any device path --
    spmv_csr2 / spmv_csr3 / spmv_gpu35 / spmv_device only run the CUDA
    library.  The device k = 1 kernel is ``spmv_device(a, x)``."""
    x = _check_x(a, x)
    y = host_row_sums(a.row_ptr, a.col_idx, a.vals, x)
    if out is not None:
        out[:] = y
        return out
    return y


def spmv_csr2(m: CsrKMatrix, x, workers: int = 1, executor=None, *,
              out=None) -> np.ndarray:
    """k = 2 SpMV, one CTA tile per run of super-rows (kernels.py:185-206).
    ``out`` (extension) receives y, e.g. a pinned host buffer."""
    if m.k != 2:
        raise ValueError(f"spmv_csr2 requires k = 2, got k = {m.k}")
    x = _check_x(m.base, x)
    return m.device().spmv_host(x, out=out)


def spmv_csr3(m: CsrKMatrix, x, workers: int = 1, executor=None, *,
              out=None) -> np.ndarray:
    """k = 3 SpMV, one CTA tile per run of super-super-rows
    (kernels.py:209-221).  Bitwise equal to the reference.  ``out``
    (extension) receives y, e.g. a pinned host buffer."""
    if m.k != 3:
        raise ValueError(f"spmv_csr3 requires k = 3, got k = {m.k}")
    x = _check_x(m.base, x)
    return m.device().spmv_host(x, out=out)


def spmv_gpu35(m: CsrKMatrix, x, dims: BlockDims, *, out=None) -> np.ndarray:
    """Streaming kernel with the GPUSpMV-3.5 summation order: row nonzeros
    strided over ``dims.x`` lanes, then the halving tree.  Bitwise equal to
    ``emulate_gpu_spmv35(m, x, dims)[0]``; no trace.  ``out`` as spmv_csr3."""
    if m.k != 3:
        raise ValueError("emulate_gpu_spmv35 requires k = 3")
    x = _check_x(m.base, x)
    if dims.x not in STRIDED_NX:
        y = emulate_gpu_spmv35(m, x, dims)[0]
        if out is not None:
            out[:] = y
            return out
        return y
    return m.device().spmv_host(x, variant=nat.CSRK_STRIDED, nx=dims.x, out=out)


def _listing(m: CsrKMatrix, x: np.ndarray, dims: BlockDims, which: int):
    n = m.base.n_rows
    dev = m.device()
    if n == 0:
        return np.zeros(0, dtype=VALUE_DTYPE), EmulationTrace.from_records([])
    xd = nat.DeviceBuffer.from_array(x)
    yd = nat.DeviceBuffer(n * 8)
    td = nat.DeviceBuffer(7 * n * 8)
    if which == 3:
        nat.call("csrk_spmv_listing3", dev.ptr, dims.x, dims.y, xd.ptr, yd.ptr, td.ptr,
                 None)
    else:
        nat.call("csrk_spmv_listing4", dev.ptr, dims.x, dims.y, dims.z, xd.ptr, yd.ptr,
                 td.ptr, None)
    y = yd.to_array(VALUE_DTYPE, n)
    t = td.to_array(np.int64, 7 * n).reshape(7, n)
    return y, EmulationTrace(*(np.ascontiguousarray(t[i]) for i in range(7)))


def emulate_gpu_spmv3(m: CsrKMatrix, x, dims: BlockDims) -> tuple:
    """PAPER Listing 3 on the device: block = super-super-row, y lanes
    stride super-rows, x lanes stride rows, serial row sums
    (kernels.py:231-261).  Returns ``(y, trace)``."""
    if m.k != 3:
        raise ValueError("emulate_gpu_spmv3 requires k = 3")
    if dims.z != 1:
        raise ValueError("the 2D mapping does not use the z dimension")
    x = _check_x(m.base, x)
    return _listing(m, x, dims, 3)


def emulate_gpu_spmv35(m: CsrKMatrix, x, dims: BlockDims) -> tuple:
    """PAPER Listing 4 on the device: z lanes stride super-rows, y lanes
    rows, x lanes the nonzeros of a row, combined by the zero-padded halving
    tree (kernels.py:284-324).  Returns ``(y, trace)``."""
    if m.k != 3:
        raise ValueError("emulate_gpu_spmv35 requires k = 3")
    x = _check_x(m.base, x)
    return _listing(m, x, dims, 4)


def check_device_vector(t, dev, length: int, name: str, dtype=None) -> None:
    """Raise ValueError unless ``t`` is a contiguous 1-D CUDA tensor on the
    matrix's device with ``length`` elements (and ``dtype`` when given):
    the kernels take raw device pointers, so a host tensor, another GPU's
    tensor, a short or a mistyped vector would be read or written out of
    bounds."""
    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.device.index != dev.device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the matrix on cuda:{dev.device}")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != 1 or t.shape[0] != length:
        raise ValueError(f"{name} must have length {length}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def spmv_device(m, x, y=None, *, dims: BlockDims | None = None, variant: str = "serial",
                stream=None):
    """Device-resident SpMV on torch CUDA tensors (float64 or float32).

    ``m`` is a CsrMatrix, CsrKMatrix or DeviceMatrix; ``x`` / ``y`` are contiguous CUDA
    tensors in the permuted index space.  ``variant`` "serial" gives the
    reference's row order, "strided" the GPUSpMV-3.5 order with
    ``dims.x`` lanes.  Launches asynchronously on ``stream`` (default: the
    current torch stream) and returns ``y``.
    """
    import torch

    base = m.base if isinstance(m, CsrKMatrix) else m
    dev = m if isinstance(m, nat.DeviceMatrix) else m.device()
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError("x must be float32 or float64")
    f32 = x.dtype == torch.float32
    check_device_vector(x, dev, base.n_cols, "x")
    if y is None:
        y = torch.empty(base.n_rows, dtype=x.dtype, device=x.device)
    else:
        check_device_vector(y, dev, base.n_rows, "y", dtype=x.dtype)
    if f32:
        dev.ensure_f32()
    nx = 1
    var = nat.CSRK_SERIAL
    if variant == "strided":
        var = nat.CSRK_STRIDED
        nx = dims.x if dims is not None else 1
    elif variant != "serial":
        raise ValueError(f"unknown variant {variant!r}")
    if stream is None:
        stream = torch.cuda.current_stream(x.device)
    dev.spmv_ptr(x.data_ptr(), y.data_ptr(), stream.cuda_stream, variant=var, nx=nx,
                 f32=f32)
    return y
