"""Full-size configurations (BASELINE.json configs C2, C3, C5) against the
digests the unmodified reference produced (tests/golden/configs.json, ~5 min
of reference Band-k each): device and host Band-k permutations and group
sizes, the device-packed CSR-k arrays, and y of the CSR-3 kernel."""

from __future__ import annotations

import time

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from conftest import digest
from paper_2203_05096_b200 import synthetic

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _matrix(spec):
    if spec["kind"] == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays(spec["shape"], spec["points"])
        return ck.CsrMatrix(n, n, rp, ci, va, _trusted=True)
    r, c, v = synthetic.irregular_triplets(spec["rows"], seed=spec.get("seed", 0))
    return ck.csr_from_arrays(spec["rows"], spec["rows"], r, c, v)


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_size_pipeline_matches_reference(name, configs_golden, capsys):
    rec = configs_golden.get(name)
    if rec is None:
        pytest.skip(f"{name} digests not generated")
    a = _matrix(rec["spec"])
    assert digest(a.row_ptr, "<u4") == rec["input"]["row_ptr"]
    assert digest(a.col_idx, "<u4") == rec["input"]["col_idx"]
    x = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
    for run in rec["runs"]:
        t0 = time.perf_counter()
        res = ck.band_k(a, 3, run["targets"], backend="device")
        t_dev = time.perf_counter() - t0
        assert digest(res.perm.fwd, "<i8") == run["fwd"]
        assert digest(res.level_group_sizes[0], "<i8") == run["sizes0"]
        assert digest(res.level_group_sizes[1], "<i8") == run["sizes1"]
        m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
        assert digest(m.base.row_ptr, "<u4") == run["base_row_ptr"]
        assert digest(m.base.col_idx, "<u4") == run["base_col_idx"]
        assert digest(m.base.vals, "<f8") == run["base_vals"]
        assert digest(m.sr_ptr, "<u4") == run["sr_ptr"]
        assert digest(m.ssr_ptr, "<u4") == run["ssr_ptr"]
        xp = ck.permute_vector(res.perm, x)
        assert digest(xp, "<f8") == run["xp"]
        y3 = ck.spmv_csr3(m, xp)
        assert digest(y3, "<f8") == run["y_csr3"]
        assert digest(ck.unpermute_vector(res.perm, y3), "<f8") == run["y_csr3_unpermuted"]
        with capsys.disabled():
            print(f"\n[{name}] device band_k {t_dev:.2f}s (reference {run['band_k_seconds']}s)")
    if name == "C2":  # the host implementation too, once
        t0 = time.perf_counter()
        res = ck.band_k(a, 3, rec["runs"][0]["targets"], backend="host")
        t_host = time.perf_counter() - t0
        assert digest(res.perm.fwd, "<i8") == rec["runs"][0]["fwd"]
        with capsys.disabled():
            print(f"[{name}] host band_k {t_host:.2f}s")
