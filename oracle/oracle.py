"""CPU oracle of the reference csrk SpMV path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, as the checker and the timed
CPU baseline; the product package never does.

Contents (each restates a reference function, file:line under
/root/reference/pkg/src/csrk/):
  spmv_serial      kernels.py:97-147   (spmv_csr_ref / _rows_spmv)       C
  spmv_grouped     kernels.py:150-221  (spmv_csr2 / spmv_csr3, threads)  C + OpenMP
  spmv_strided     kernels.py:264-324  (emulate_gpu_spmv35 arithmetic)   C
  permute_symmetric format.py:318-344  (_permute_symmetric)              C
  gather           format.py:396-409   (permute_vector / unpermute)      C
  group_pointers   format.py:383-388   (pack_csrk prefix sums)           numpy
  abs_row_dot      |A||x| for the scaled error bound   C

Pinning: tests/test_oracle.py checks every function against the golden
vectors that tests/golden/make_golden.py produced by running the unmodified
reference.  The Band-k reordering has no restatement here: the product's
native Band-k is compared directly with the reference's permutations
(tests/golden/small_cases.npz, configs.json digests).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None

_U32 = C.POINTER(C.c_uint32)
_I64 = C.POINTER(C.c_int64)
_F64 = C.POINTER(C.c_double)


def build() -> str:
    src = os.path.join(HERE, "csrk_oracle.c")
    if not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        lib.oracle_spmv_serial.argtypes = [C.c_int64, _U32, _U32, _F64, _F64, _F64]
        lib.oracle_spmv_grouped.argtypes = [C.c_int64, _I64, _U32, _U32, _F64, _F64,
                                            _F64, C.c_int]
        lib.oracle_spmv_strided.argtypes = [C.c_int64, _U32, _U32, _F64, _F64, _F64,
                                            C.c_int]
        lib.oracle_permute_symmetric.argtypes = [C.c_int64, _U32, _U32, _F64, _I64,
                                                 _I64, _U32, _U32, _F64]
        lib.oracle_gather.argtypes = [C.c_int64, _F64, _I64, _F64]
        lib.oracle_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(_U32)


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_I64)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_F64)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def spmv_serial(row_ptr, col_idx, vals, x) -> np.ndarray:
    rp, prp = _u32(row_ptr)
    ci, pci = _u32(col_idx)
    va, pva = _f64(vals)
    xx, px = _f64(x)
    y = np.zeros(len(rp) - 1)
    _load().oracle_spmv_serial(len(rp) - 1, prp, pci, pva, px, y.ctypes.data_as(_F64))
    return y


def spmv_grouped(group_rows, row_ptr, col_idx, vals, x, workers=1) -> np.ndarray:
    gr, pgr = _i64(group_rows)
    rp, prp = _u32(row_ptr)
    ci, pci = _u32(col_idx)
    va, pva = _f64(vals)
    xx, px = _f64(x)
    y = np.zeros(len(rp) - 1)
    _load().oracle_spmv_grouped(len(gr) - 1, pgr, prp, pci, pva, px,
                                y.ctypes.data_as(_F64), int(workers))
    return y


def csr3_group_rows(sr_ptr, ssr_ptr) -> np.ndarray:
    """Row offsets of the super-super-rows, sr_ptr[ssr_ptr] (kernels.py:220)."""
    return np.asarray(sr_ptr, dtype=np.int64)[np.asarray(ssr_ptr, dtype=np.int64)]


def spmv_strided(row_ptr, col_idx, vals, x, nx) -> np.ndarray:
    rp, prp = _u32(row_ptr)
    ci, pci = _u32(col_idx)
    va, pva = _f64(vals)
    xx, px = _f64(x)
    y = np.zeros(len(rp) - 1)
    _load().oracle_spmv_strided(len(rp) - 1, prp, pci, pva, px, y.ctypes.data_as(_F64),
                                int(nx))
    return y


def permute_symmetric(row_ptr, col_idx, vals, fwd, inv):
    rp, prp = _u32(row_ptr)
    ci, pci = _u32(col_idx)
    va, pva = _f64(vals)
    f, pf = _i64(fwd)
    iv, piv = _i64(inv)
    n = len(rp) - 1
    out_ptr = np.zeros(n + 1, dtype=np.uint32)
    out_cols = np.zeros(len(ci), dtype=np.uint32)
    out_vals = np.zeros(len(ci))
    _load().oracle_permute_symmetric(n, prp, pci, pva, pf, piv,
                                     out_ptr.ctypes.data_as(_U32),
                                     out_cols.ctypes.data_as(_U32),
                                     out_vals.ctypes.data_as(_F64))
    return out_ptr, out_cols, out_vals


def gather(x, idx) -> np.ndarray:
    xx, px = _f64(x)
    ii, pii = _i64(idx)
    out = np.zeros(len(ii))
    _load().oracle_gather(len(ii), px, pii, out.ctypes.data_as(_F64))
    return out


def group_pointers(sizes) -> np.ndarray:
    """pack_csrk's pointer arrays: 0 followed by the running sum (uint32)."""
    s = np.asarray(sizes, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(s)]).astype(np.uint32)


def abs_row_dot(row_ptr, col_idx, vals, x) -> np.ndarray:
    """(|A||x|)_i, the scale of the error bound of SURVEY.md §8(c)(3)."""
    return spmv_serial(row_ptr, col_idx, np.abs(np.asarray(vals, dtype=np.float64)),
                       np.abs(np.asarray(x, dtype=np.float64)))
