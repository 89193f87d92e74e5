"""The C-ABI library loads on a CPU-only machine and exports every symbol
include/csrk.h declares; host-side entry points report errors with the
reference's messages."""

from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "csrk.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(csrk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2203_05096_b200 import _native
    lib = C.CDLL(_native.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name
    # the ctypes binding covers the whole header
    assert set(names) == set(_native.EXPORTED)


def test_abi_version_and_error_channel():
    from paper_2203_05096_b200 import _native
    lib = _native.lib()
    assert lib.csrk_abi_version() == 1
    out = C.c_void_p()
    rp = np.array([0, 1], dtype=np.uint32)
    ci = np.array([0], dtype=np.uint32)
    targets = np.array([2.0, 2.0, 2.0])
    rc = lib.csrk_band_k(1, _native.u32p(rp), _native.u32p(ci), 4,
                         _native.f64p(targets), C.byref(out))
    assert rc == _native.CSRK_EINVAL
    assert b"k must be 2 or 3" in lib.csrk_last_error()
    with pytest.raises(ValueError, match="k must be 2 or 3"):
        _native.check(rc)


def test_pack_validation_happens_before_device_work():
    """csrk_pack rejects bad group sizes without touching a GPU."""
    from paper_2203_05096_b200 import _native
    lib = _native.lib()
    n = 4
    rp = np.array([0, 1, 2, 3, 4], dtype=np.uint32)
    ci = np.arange(4, dtype=np.uint32)
    va = np.ones(4)
    fwd = np.arange(4, dtype=np.int64)
    s1 = np.array([2, 1], dtype=np.int64)
    out = C.c_void_p()
    rc = lib.csrk_pack(0, n, 4, _native.u32p(rp), _native.u32p(ci), _native.f64p(va),
                       _native.i64p(fwd), _native.i64p(fwd), 1, 2, _native.i64p(s1), 0,
                       None, C.byref(out))
    assert rc == _native.CSRK_EINVAL
    assert b"level 1 group sizes sum to 3, expected 4" in lib.csrk_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2203_05096_b200 import _native
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "absent.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.lib()


@pytest.mark.gpu
def test_spmv_kernels_launch_first():
    """The hot kernels run through the library before anything else of the
    GPU suite (csrk_stream_kernel in both orders, long_rows_kernel beside
    it), checked against the oracle -- no Band-k on this path."""
    import numpy as np

    import paper_2203_05096_b200 as ck
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    n = 20000
    lens = rng.integers(0, 16, n)
    lens[[5, 9000]] = (700, 3000)
    rows = np.repeat(np.arange(n), lens)
    a = ck.csr_from_arrays(n, n, rows, rng.integers(0, n, len(rows)),
                           rng.uniform(-1, 1, len(rows)))
    m = ck.pack_csrk(a, ck.Permutation.identity(n), [[1] * n, [n]])
    x = rng.uniform(-1, 1, n)
    assert np.array_equal(ck.spmv_csr3(m, x), O.spmv_serial(a.row_ptr, a.col_idx, a.vals, x))
    assert np.array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(8, 1, 1)),
                          O.spmv_strided(a.row_ptr, a.col_idx, a.vals, x, 8))
    assert m.device().plan()["n_long"] == 2
