"""Deterministic synthetic matrices for the BASELINE.json configurations.

The configs (BASELINE.json ``configs``; SURVEY.md §8(d) "Synthetic inputs")
are grid Laplacians in natural lexicographic order (x fastest) and one
irregular random-row-length matrix.  Stencil matrices are emitted directly in
canonical CSR form (columns strictly increasing, no duplicates), which is
exactly what ``csr_from_arrays`` (reference format.py:233-284) returns for the
same triplets; the golden script checks that equivalence.

Stencil values follow the reference's own grid fixtures: diagonal = number of
neighbours of an interior point (4, 6 or 26), off-diagonals -1
(pkg/tests/oracles.py:94-110, pkg/tests/test_acceptance.py:219-233).  With
``values="uniform"`` the values are instead U[0.5, 1.5) from
``numpy.random.default_rng(seed)`` in entry order.
"""

from __future__ import annotations

import itertools

import numpy as np

__all__ = [
    "CONFIGS",
    "stencil_arrays",
    "irregular_triplets",
    "config_arrays",
    "config_x",
]

# name -> (kind, shape or rows, points); C4 is the CG-loop config.
CONFIGS = {
    "C1": ("stencil", (1000, 1000), 5),
    "C2": ("stencil", (256, 256, 256), 7),
    "C3": ("stencil", (192, 192, 192), 27),
    "C4": ("stencil", (512, 512, 512), 7),
    "C5": ("irregular", 5_000_000, None),
}


def _offsets(ndim: int, points: int) -> list:
    """Stencil offsets as coordinate tuples, slowest axis first."""
    if points == 2 * ndim + 1:
        offs = [tuple(0 for _ in range(ndim))]
        for axis in range(ndim):
            for step in (-1, 1):
                o = [0] * ndim
                o[axis] = step
                offs.append(tuple(o))
    elif points == 3 ** ndim:
        offs = list(itertools.product((-1, 0, 1), repeat=ndim))
    else:
        raise ValueError(f"unsupported stencil: {points} points in {ndim}D")
    return offs


def stencil_arrays(shape, points: int, values: str = "laplacian", seed: int = 0,
                   index_dtype=np.uint32):
    """Canonical CSR arrays ``(n, row_ptr, col_idx, vals)`` of a grid stencil.

    ``shape`` lists grid extents slowest axis first (``(ny, nx)`` or
    ``(nz, ny, nx)``); row i = (z*ny + y)*nx + x.
    """
    shape = tuple(int(s) for s in shape)
    ndim = len(shape)
    n = int(np.prod(shape))
    offs = _offsets(ndim, points)
    strides = [int(np.prod(shape[a + 1:])) for a in range(ndim)]
    lin = sorted((sum(o[a] * strides[a] for a in range(ndim)), o) for o in offs)
    diag = float(len(offs) - 1)
    # Per-axis validity is separable: an offset is valid for a row when every
    # coordinate stays inside the grid.  Work in row chunks to bound memory.
    counts = np.zeros(n, dtype=np.int64)
    chunk = 1 << 22
    coord_cache = {}

    def coords(lo, hi):
        idx = np.arange(lo, hi, dtype=np.int64)
        out = []
        for a in range(ndim):
            out.append((idx // strides[a]) % shape[a])
        return idx, out

    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        idx, cs = coords(lo, hi)
        c = np.zeros(hi - lo, dtype=np.int64)
        for _, o in lin:
            ok = np.ones(hi - lo, dtype=bool)
            for a in range(ndim):
                if o[a] < 0:
                    ok &= cs[a] >= -o[a]
                elif o[a] > 0:
                    ok &= cs[a] < shape[a] - o[a]
            c += ok
        counts[lo:hi] = c
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col_idx = np.empty(nnz, dtype=index_dtype)
    vals = np.empty(nnz, dtype=np.float64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        idx, cs = coords(lo, hi)
        m = hi - lo
        cols2 = np.empty((m, len(lin)), dtype=np.int64)
        keep = np.empty((m, len(lin)), dtype=bool)
        vals2 = np.empty((m, len(lin)), dtype=np.float64)
        for j, (d, o) in enumerate(lin):
            ok = np.ones(m, dtype=bool)
            for a in range(ndim):
                if o[a] < 0:
                    ok &= cs[a] >= -o[a]
                elif o[a] > 0:
                    ok &= cs[a] < shape[a] - o[a]
            keep[:, j] = ok
            cols2[:, j] = idx + d
            vals2[:, j] = diag if d == 0 else -1.0
        p0, p1 = int(row_ptr[lo]), int(row_ptr[hi])
        col_idx[p0:p1] = cols2[keep]
        vals[p0:p1] = vals2[keep]
    if values == "uniform":
        vals = np.random.default_rng(seed).uniform(0.5, 1.5, nnz)
    elif values != "laplacian":
        raise ValueError(f"unknown value set {values!r}")
    return n, row_ptr.astype(index_dtype), col_idx, vals


def irregular_triplets(n_rows: int = 5_000_000, seed: int = 0,
                       max_len: int = 19, reach: int = 65_536):
    """COO triplets of the irregular config (SURVEY.md §8(d) "C5").

    Row length L ~ U{1..max_len}; the first entry of every row is the
    diagonal, the other L-1 columns are the row index plus an offset
    ~ U[-reach, reach], clipped into [0, n).  Duplicate coordinates are left
    in place for ``csr_from_arrays`` to merge.  Values ~ U[0.5, 1.5).
    """
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_len + 1, n_rows)
    total = int(lens.sum())
    rows = np.repeat(np.arange(n_rows, dtype=np.int64), lens)
    offs = rng.integers(-reach, reach + 1, total)
    starts = np.zeros(n_rows, dtype=np.int64)
    np.cumsum(lens[:-1], out=starts[1:])
    offs[starts] = 0
    cols = np.clip(rows + offs, 0, n_rows - 1)
    vals = rng.uniform(0.5, 1.5, total)
    return rows, cols, vals


def config_arrays(name: str, values: str = "laplacian"):
    """CSR arrays of a named config; C5 goes through ``csr_from_arrays``."""
    kind, shape, points = CONFIGS[name]
    if kind == "stencil":
        from . import _native as nat
        if values == "laplacian" and nat.device_count() > 0:
            # generated in HBM (bitwise the host generator) and downloaded
            rp, ci, va, _, _ = device_stencil(shape, points).download()
            return len(rp) - 1, rp, ci, va
        return stencil_arrays(shape, points, values=values)
    from .format import csr_from_arrays
    rows, cols, vals = irregular_triplets(shape)
    a = csr_from_arrays(shape, shape, rows, cols, vals)
    return a.n_rows, a.row_ptr, a.col_idx, a.vals


def config_x(n: int, seed: int = 0) -> np.ndarray:
    """The dense input vector ``run_benchmark`` draws (reference
    bench.py:270-271): ``default_rng(seed).uniform(-1, 1, n)``."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def device_stencil(shape, points: int, device=None):
    """Generate a stencil matrix directly in HBM (csrk_stencil, csrc/construct.cu):
    canonical CSR, natural order, Laplacian values; returns a k = 1
    ``_native.DeviceMatrix``.  Bitwise equal to :func:`stencil_arrays`."""
    import ctypes as C

    from . import _native as nat

    dims = [int(s) for s in shape]
    if len(dims) == 2:
        dims = [1] + dims
    out = C.c_void_p()
    nat.call("csrk_stencil", nat.current_device() if device is None else device,
             dims[0], dims[1], dims[2], int(points), C.byref(out))
    return nat.DeviceMatrix(out)


def device_slab(shape, points: int, z0: int, z1: int, device=None):
    """Rows of planes [z0, z1) of a 3D stencil generated in HBM
    (csrk_stencil_slab): natural order, columns numbered from plane
    max(z0 - 1, 0), so x is [lower halo plane | own planes | upper halo
    plane].  Returns a k = 1 ``_native.DeviceMatrix``; its rows equal rows
    [z0 * ny * nx, z1 * ny * nx) of :func:`device_stencil` with the columns
    shifted by ``max(z0 - 1, 0) * ny * nx``."""
    import ctypes as C

    from . import _native as nat

    nz, ny, nx = (int(s) for s in shape)
    out = C.c_void_p()
    nat.call("csrk_stencil_slab", nat.current_device() if device is None else device,
             nz, ny, nx, int(points), int(z0), int(z1), C.byref(out))
    return nat.DeviceMatrix(out)
