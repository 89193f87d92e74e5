"""CSR and CSR-k containers with device residency.

Drop-in for the reference's ``csrk.format`` (pkg/src/csrk/format.py).  The
host objects keep the reference's storage contract -- uint32 indices, float64
values, int64 permutations, frozen arrays, identical validation messages --
and additionally carry a lazily created device copy (``_native.DeviceMatrix``)
so repeated SpMVs run on resident HBM data (PAPER.md:643-644 times kernels on
pre-resident data).

What runs where:
  * container validation and COO assembly (``csr_from_arrays``) -- host, as
    input staging;
  * ``pack_csrk`` -- the symmetric permutation P.A.P^T, the per-row column
    sort and the group pointer prefix sums run on the device
    (``csrk_pack``, csrc/construct.cu); the packed matrix stays resident;
  * ``permute_vector`` / ``unpermute_vector`` -- device gathers.
"""

from __future__ import annotations

import ctypes
from typing import Iterable, Sequence

import numpy as np

from . import _native as nat

__all__ = [
    "INDEX_DTYPE",
    "VALUE_DTYPE",
    "MAX_NNZ",
    "CsrMatrix",
    "CsrKMatrix",
    "Permutation",
    "build_csr",
    "csr_from_arrays",
    "pack_csrk",
    "permute_vector",
    "unpermute_vector",
]

INDEX_DTYPE = np.uint32          # format.py:32
VALUE_DTYPE = np.float64         # format.py:33
MAX_NNZ = 2 ** 31 - 1            # format.py:37


def _readonly(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


class _Frozen:
    """Attribute assignment is an error after construction (the reference
    uses frozen dataclasses).  Internal caches go through _cache()."""

    __slots__ = ()

    def __setattr__(self, name, value):
        raise AttributeError(f"{type(self).__name__} is immutable")

    def __delattr__(self, name):
        raise AttributeError(f"{type(self).__name__} is immutable")

    def _set(self, name, value):
        object.__setattr__(self, name, value)


class CsrMatrix(_Frozen):
    """Compressed sparse rows: uint32 ``row_ptr`` (n_rows + 1) and
    ``col_idx`` (nnz), float64 ``vals``; columns strictly increase within a
    row.  Mirrors reference format.py:45-113 (validation 71-98)."""

    __slots__ = ("n_rows", "n_cols", "row_ptr", "col_idx", "vals", "_dev")

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, vals, *, _trusted=False):
        n_rows, n_cols = int(n_rows), int(n_cols)
        if n_rows < 0 or n_cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        rp = np.array(row_ptr, dtype=INDEX_DTYPE, copy=True)
        ci = np.array(col_idx, dtype=INDEX_DTYPE, copy=True)
        va = np.array(vals, dtype=VALUE_DTYPE, copy=True)
        if not _trusted:
            _check_csr(n_rows, n_cols, rp, ci, va)
        self._set("n_rows", n_rows)
        self._set("n_cols", n_cols)
        self._set("row_ptr", _readonly(rp))
        self._set("col_idx", _readonly(ci))
        self._set("vals", _readonly(va))
        self._set("_dev", None)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def row_nnz(self) -> np.ndarray:
        """Stored entries per row (int64)."""
        return np.diff(self.row_ptr.astype(np.int64))

    def device(self) -> nat.DeviceMatrix:
        """The resident device copy (uploaded on first use, k = 1 CSR)."""
        if self._dev is None:
            self._set("_dev", nat.DeviceMatrix.upload(
                self.row_ptr, self.col_idx, self.vals, self.n_rows, self.n_cols, k=1))
        return self._dev

    def __repr__(self) -> str:
        return f"CsrMatrix(n_rows={self.n_rows}, n_cols={self.n_cols}, nnz={self.nnz})"


def _check_csr(n_rows, n_cols, rp, ci, va):
    if rp.ndim != 1 or rp.shape[0] != n_rows + 1:
        raise ValueError("row_ptr must have length n_rows + 1")
    if rp[0] != 0:
        raise ValueError("row_ptr[0] must be 0")
    steps = np.diff(rp.astype(np.int64))
    if steps.size and steps.min() < 0:
        raise ValueError("row_ptr must be non-decreasing")
    nnz = int(rp[-1])
    if nnz > MAX_NNZ:
        raise ValueError(f"nnz {nnz} exceeds the 32-bit index limit {MAX_NNZ}")
    if ci.shape[0] != nnz or va.shape[0] != nnz:
        raise ValueError("col_idx and vals must have length row_ptr[-1]")
    if nnz == 0:
        return
    if int(ci.max()) >= n_cols:
        raise ValueError("column index out of range")
    # consecutive entries of the same row must strictly increase
    same_row = np.ones(nnz - 1, dtype=bool)
    row_starts = rp[1:-1].astype(np.int64)
    row_starts = row_starts[(row_starts > 0) & (row_starts < nnz)]
    same_row[row_starts - 1] = False
    if np.any(np.diff(ci.astype(np.int64))[same_row] <= 0):
        raise ValueError("col_idx must be strictly increasing within each row")


class Permutation(_Frozen):
    """Row bijection stored both ways: ``fwd[old] = new``, ``inv[new] = old``
    (int64).  Mirrors reference format.py:116-161."""

    __slots__ = ("fwd", "inv", "_dev_inv", "_dev_fwd")

    def __init__(self, fwd, inv, *, _trusted=False):
        f = np.array(fwd, dtype=np.int64, copy=True)
        i = np.array(inv, dtype=np.int64, copy=True)
        if not _trusted:
            n = f.shape[0]
            if i.shape[0] != n:
                raise ValueError("fwd and inv must have equal length")
            if n and (f.min() < 0 or f.max() >= n):
                raise ValueError("permutation entries out of range")
            ar = np.arange(n)
            if n and (i.min() < 0 or i.max() >= n or np.any(f[i] != ar)
                      or np.any(i[f] != ar)):
                raise ValueError("fwd and inv are not mutually inverse bijections")
        self._set("fwd", _readonly(f))
        self._set("inv", _readonly(i))
        self._set("_dev_inv", None)
        self._set("_dev_fwd", None)

    @classmethod
    def from_forward(cls, fwd: Sequence[int]) -> "Permutation":
        f = np.asarray(fwd, dtype=np.int64)
        n = f.shape[0]
        if n and (f.min() < 0 or f.max() >= n):
            raise ValueError("permutation entries out of range")
        inv = np.empty(n, dtype=np.int64)
        inv[f] = np.arange(n, dtype=np.int64)
        return cls(f, inv)

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        ar = np.arange(int(n), dtype=np.int64)
        return cls(ar, ar, _trusted=True)

    def device_index(self, which: str) -> nat.DeviceBuffer:
        """Resident copy of ``inv`` or ``fwd`` for device gathers."""
        slot = "_dev_inv" if which == "inv" else "_dev_fwd"
        buf = getattr(self, slot)
        if buf is None:
            buf = nat.DeviceBuffer.from_array(self.inv if which == "inv" else self.fwd)
            self._set(slot, buf)
        return buf

    def __len__(self) -> int:
        return int(self.fwd.shape[0])

    def __repr__(self) -> str:
        return f"Permutation(n={len(self)})"


class CsrKMatrix(_Frozen):
    """P.A.P^T in CSR form plus k - 1 group pointer arrays: ``sr_ptr``
    (rows per super-row) and for k = 3 ``ssr_ptr`` (super-rows per
    super-super-row).  Mirrors reference format.py:164-230."""

    __slots__ = ("base", "k", "group_ptrs", "perm", "_dev")

    def __init__(self, base: CsrMatrix, k: int, group_ptrs, perm: Permutation, *,
                 _trusted=False, _device=None):
        if k not in (2, 3):
            raise ValueError("k must be 2 or 3")
        ptrs = tuple(_readonly(np.array(p, dtype=INDEX_DTYPE, copy=True))
                     for p in group_ptrs)
        if len(ptrs) != k - 1:
            raise ValueError("expected k - 1 grouping pointer arrays")
        if not _trusted:
            below = base.n_rows
            for level, p in enumerate(ptrs, start=1):
                if p.shape[0] < 1 or p[0] != 0:
                    raise ValueError(f"level {level} pointer array must start at 0")
                if np.any(np.diff(p.astype(np.int64)) <= 0):
                    raise ValueError(
                        f"level {level} pointer array must be strictly increasing")
                if int(p[-1]) != below:
                    raise ValueError(
                        f"level {level} pointer array must end at {below}, got {int(p[-1])}")
                below = p.shape[0] - 1
        if len(perm) != base.n_rows:
            raise ValueError("permutation length must match n_rows")
        self._set("base", base)
        self._set("k", int(k))
        self._set("group_ptrs", ptrs)
        self._set("perm", perm)
        self._set("_dev", _device)

    @property
    def sr_ptr(self) -> np.ndarray:
        return self.group_ptrs[0]

    @property
    def ssr_ptr(self) -> np.ndarray:
        if self.k != 3:
            raise AttributeError("ssr_ptr exists only for k = 3")
        return self.group_ptrs[1]

    @property
    def num_super_rows(self) -> int:
        return self.group_ptrs[0].shape[0] - 1

    @property
    def num_ssr(self) -> int:
        return self.ssr_ptr.shape[0] - 1

    def as_csr(self) -> CsrMatrix:
        """The base CSR arrays (shared, no copy)."""
        return self.base

    def device(self) -> nat.DeviceMatrix:
        """Resident CSR-k copy (present after pack_csrk, else uploaded)."""
        if self._dev is None:
            b = self.base
            self._set("_dev", nat.DeviceMatrix.upload(
                b.row_ptr, b.col_idx, b.vals, b.n_rows, b.n_cols, k=self.k,
                sr_ptr=self.group_ptrs[0],
                ssr_ptr=self.group_ptrs[1] if self.k == 3 else None))
        return self._dev

    def __repr__(self) -> str:
        return (f"CsrKMatrix(k={self.k}, n_rows={self.base.n_rows}, "
                f"nnz={self.base.nnz}, num_super_rows={self.num_super_rows})")


DEVICE_COO_MIN = 1 << 16  # triplet count from which csr_from_arrays runs on the GPU


def csr_from_arrays(n_rows: int, n_cols: int, rows, cols, vals) -> CsrMatrix:
    """Canonical CSR from coordinate triplets in any order; duplicate
    coordinates are summed in their input order (reference
    format.py:233-284).  Large inputs are assembled on the GPU
    (csrk_coo_to_csr), bit-identical to the host restatement below."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(vals, dtype=VALUE_DTYPE)
    count = r.shape[0]
    if c.shape[0] != count or v.shape[0] != count:
        raise ValueError("coordinate arrays must have equal length")
    if count > MAX_NNZ:
        raise ValueError(f"entry count {count} exceeds the 32-bit index limit")
    for name, arr, bound in (("row", r, n_rows), ("column", c, n_cols)):
        bad = np.flatnonzero((arr < 0) | (arr >= bound))
        if bad.size:
            p = int(bad[0])
            raise ValueError(
                f"triplet {p}: {name} index {int(arr[p])} out of range [0, {bound})")
    if count == 0:
        return CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, dtype=np.int64),
                         np.empty(0, dtype=np.int64), np.empty(0), _trusted=True)
    if count >= DEVICE_COO_MIN and nat.device_count() > 0:
        # on the GPU: stable radix sort + duplicate runs summed in numpy's
        # reduceat order (csrk_coo_to_csr); the result keeps its device copy
        out = ctypes.c_void_p()
        r, c, v = (np.ascontiguousarray(t) for t in (r, c, v))
        nat.call("csrk_coo_to_csr", nat.current_device(), n_rows, n_cols, count,
                 nat.i64p(r), nat.i64p(c), nat.f64p(v), ctypes.byref(out))
        dev = nat.DeviceMatrix(out)
        rp, ci, va, _, _ = dev.download()
        m = CsrMatrix(n_rows, n_cols, rp, ci, va, _trusted=True)
        m._set("_dev", dev)
        return m
    # stable order by (row, col); equal coordinates keep their input order
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    head = np.empty(count, dtype=bool)
    head[0] = True
    np.not_equal(r[1:], r[:-1], out=head[1:])
    head[1:] |= c[1:] != c[:-1]
    starts = np.flatnonzero(head)
    summed = np.add.reduceat(v, starts)
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(r[starts], minlength=n_rows))
    return CsrMatrix(n_rows, n_cols, ptr, c[starts], summed, _trusted=True)


def build_csr(n_rows: int, n_cols: int, triplets: Iterable[tuple]) -> CsrMatrix:
    """Canonical CSR from an iterable of (row, col, value) triplets."""
    data = list(triplets)
    rows = np.array([t[0] for t in data], dtype=np.int64)
    cols = np.array([t[1] for t in data], dtype=np.int64)
    vals = np.array([t[2] for t in data], dtype=VALUE_DTYPE)
    return csr_from_arrays(n_rows, n_cols, rows, cols, vals)


def _level_sizes(groups, n_rows):
    if len(groups) not in (1, 2):
        raise ValueError("groups must hold 1 or 2 levels (k = 2 or 3)")
    out = []
    below = n_rows
    for level, sizes in enumerate(groups, start=1):
        s = np.asarray(sizes, dtype=np.int64).reshape(-1)
        if s.shape[0] == 0 or np.any(s < 1):
            raise ValueError(f"level {level} group sizes must be positive")
        total = int(s.sum())
        if total != below:
            raise ValueError(f"level {level} group sizes sum to {total}, expected {below}")
        out.append(np.ascontiguousarray(s))
        below = s.shape[0]
    return out


def pack_csrk(a: CsrMatrix, perm: Permutation, groups: Sequence[Sequence[int]],
              *, download: bool = True) -> CsrKMatrix:
    """Assemble CSR-k from a permutation and per-level group sizes
    (reference format.py:347-393).  The permutation P.A.P^T, the per-row
    column sort and the pointer prefix sums run on the device; the result
    stays resident for SpMV and (by default) is copied back so the host
    arrays match the reference's objects exactly."""
    if a.n_rows != a.n_cols:
        raise ValueError("CSR-k packing requires a square matrix")
    if len(groups) not in (1, 2):
        raise ValueError("groups must hold 1 or 2 levels (k = 2 or 3)")
    if len(perm) != a.n_rows:
        raise ValueError("permutation length must match n_rows")
    sizes = _level_sizes(groups, a.n_rows)
    k = len(sizes) + 1
    import ctypes as C
    out = C.c_void_p()
    s2 = sizes[1] if k == 3 else np.zeros(1, dtype=np.int64)
    nat.call("csrk_pack", nat.current_device(), a.n_rows, a.nnz,
             nat.u32p(a.row_ptr), nat.u32p(a.col_idx), nat.f64p(a.vals),
             nat.i64p(perm.fwd), nat.i64p(perm.inv), k - 1, sizes[0].shape[0],
             nat.i64p(sizes[0]), s2.shape[0] if k == 3 else 0, nat.i64p(s2),
             C.byref(out))
    dev = nat.DeviceMatrix(out)
    if download:
        rp, ci, va, sp, ssp = dev.download()
    else:  # pointers only; base arrays stay on the device
        rp, ci, va = (np.zeros(a.n_rows + 1, dtype=np.uint32), np.zeros(0, np.uint32),
                      np.zeros(0))
        sp = np.concatenate([[0], np.cumsum(sizes[0])])
        ssp = np.concatenate([[0], np.cumsum(sizes[1])]) if k == 3 else None
    base = CsrMatrix(a.n_rows, a.n_cols, rp, ci, va, _trusted=True)
    ptrs = (sp,) if k == 2 else (sp, ssp)
    return CsrKMatrix(base, k, ptrs, perm, _trusted=True, _device=dev)


def _gather(x: np.ndarray, p: Permutation, which: str) -> np.ndarray:
    n = len(p)
    out = nat.DeviceBuffer(max(8, n * 8))
    if n == 0:
        return np.empty(0, dtype=VALUE_DTYPE)
    xin = nat.DeviceBuffer.from_array(np.ascontiguousarray(x, dtype=VALUE_DTYPE))
    idx = p.device_index(which)
    nat.call("csrk_gather_f64", n, xin.ptr, idx.ptr, out.ptr, None)
    return out.to_array(VALUE_DTYPE, n)


def permute_vector(p: Permutation, x) -> np.ndarray:
    """Vector into the permuted index space: ``out[fwd[i]] = x[i]``
    (reference format.py:396-401); a device gather through ``p.inv``."""
    x = np.asarray(x, dtype=VALUE_DTYPE)
    if x.shape[0] != len(p):
        raise ValueError(f"vector length {x.shape[0]} does not match permutation {len(p)}")
    return _gather(x, p, "inv")


def unpermute_vector(p: Permutation, y) -> np.ndarray:
    """Inverse of permute_vector: ``out[i] = y[fwd[i]]`` (format.py:404-409)."""
    y = np.asarray(y, dtype=VALUE_DTYPE)
    if y.shape[0] != len(p):
        raise ValueError(f"vector length {y.shape[0]} does not match permutation {len(p)}")
    return _gather(y, p, "fwd")
