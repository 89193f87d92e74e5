"""Shared fixtures.  ``-m gpu`` tests need a B200 (run through gpurun);
everything else runs on a CPU-only machine."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: full-size configurations")


def has_gpu() -> bool:
    try:
        from paper_2203_05096_b200 import _native
        return _native.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def digest(arr, dtype) -> str:
    a = np.ascontiguousarray(np.asarray(arr).astype(dtype, copy=False))
    return hashlib.sha256(a.tobytes()).hexdigest()


class Golden:
    """Accessor over tests/golden/small_cases.npz (written by
    tests/golden/make_golden.py from the unmodified reference)."""

    def __init__(self):
        self.z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
        self.names = [str(n) for n in self.z["names"]]

    def __getitem__(self, key):
        return self.z[key]

    def has(self, key) -> bool:
        return key in self.z.files

    def csr(self, name):
        from paper_2203_05096_b200 import CsrMatrix
        shape = self.z[f"{name}/shape"]
        return CsrMatrix(int(shape[0]), int(shape[1]), self.z[f"{name}/row_ptr"],
                         self.z[f"{name}/col_idx"], self.z[f"{name}/vals"])


BANDK_TAGS = (("k2_4", 2, [4]), ("k3_4_2", 3, [4, 2]), ("k3_2_3", 3, [2, 3]),
              ("k3_8_4", 3, [8, 4]))


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def configs_golden():
    path = os.path.join(GOLDEN, "configs.json")
    with open(path) as fh:
        return json.load(fh)


def tridiagonal(n: int, seed: int = 0):
    """pkg/tests/conftest.py:19-29: n x n tridiagonal, values U[0.5, 1.5)."""
    from paper_2203_05096_b200 import csr_from_arrays
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
    vals = rng.uniform(0.5, 1.5, len(rows))
    return csr_from_arrays(n, n, np.array(rows), np.array(cols), vals)


def random_csr(rng, n_rows, n_cols, density, value_low=0.5, value_high=1.5):
    """pkg/tests/conftest.py:32-43: unique random positions."""
    from paper_2203_05096_b200 import csr_from_arrays
    want = min(max(0, int(round(density * n_rows * n_cols))), n_rows * n_cols)
    flat = rng.choice(n_rows * n_cols, size=want, replace=False)
    return csr_from_arrays(n_rows, n_cols, (flat // n_cols).astype(np.int64),
                           (flat % n_cols).astype(np.int64),
                           rng.uniform(value_low, value_high, size=want))
