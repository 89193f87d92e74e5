"""Pin the CPU oracle to the reference: every oracle function reproduces the
golden vectors that the unmodified reference produced (tests/golden)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import BANDK_TAGS, digest
from oracle import oracle as O

EMU35_DIMS = [(4, 8, 12), (8, 8, 8), (16, 8, 4), (2, 2, 2), (3, 5, 2), (1, 3, 4), (32, 2, 2)]


def test_oracle_spmv_serial_matches_reference(golden):
    for name in golden.names:
        a = golden.csr(name)
        for xs in ("pos", "sgn"):
            y = O.spmv_serial(a.row_ptr, a.col_idx, a.vals, golden[f"{name}/x_{xs}"])
            np.testing.assert_array_equal(y, golden[f"{name}/y_ref_{xs}"], err_msg=name)


def _packed(golden, name, tag):
    p = f"{name}/{tag}"
    ptrs = [golden[f"{p}/ptr{lv}"] for lv in range(2) if golden.has(f"{p}/ptr{lv}")]
    return (golden[f"{p}/base_row_ptr"], golden[f"{p}/base_col_idx"],
            golden[f"{p}/base_vals"], ptrs)


def test_oracle_grouped_kernels_match_reference(golden):
    for name in golden.names:
        for tag, k, _ in BANDK_TAGS:
            rp, ci, va, ptrs = _packed(golden, name, tag)
            fwd = golden[f"{name}/{tag}/fwd"]
            inv = np.empty_like(fwd)
            inv[fwd] = np.arange(len(fwd))
            for xs in ("pos", "sgn"):
                xp = O.gather(golden[f"{name}/x_{xs}"], inv)
                if k == 2:
                    rows = ptrs[0].astype(np.int64)
                    want = golden[f"{name}/{tag}/y_csr2_{xs}"]
                else:
                    rows = O.csr3_group_rows(ptrs[0], ptrs[1])
                    want = golden[f"{name}/{tag}/y_csr3_{xs}"]
                for workers in (1, 3):
                    y = O.spmv_grouped(rows, rp, ci, va, xp, workers)
                    np.testing.assert_array_equal(y, want, err_msg=f"{name} {tag}")


def test_oracle_strided_matches_emulate_gpu_spmv35(golden):
    for name in golden.names:
        tag = "k3_4_2"
        rp, ci, va, _ = _packed(golden, name, tag)
        fwd = golden[f"{name}/{tag}/fwd"]
        inv = np.argsort(fwd)
        for xs in ("pos", "sgn"):
            xp = O.gather(golden[f"{name}/x_{xs}"], inv)
            for d in EMU35_DIMS:
                key = f"{name}/{tag}/y_emu35_{'x'.join(map(str, d))}_{xs}"
                if not golden.has(key):
                    continue
                y = O.spmv_strided(rp, ci, va, xp, d[0])
                np.testing.assert_array_equal(y, golden[key], err_msg=f"{name} {d}")


def test_oracle_pack_matches_reference(golden):
    for name in golden.names:
        a = golden.csr(name)
        for tag, k, _ in BANDK_TAGS:
            fwd = golden[f"{name}/{tag}/fwd"]
            inv = np.argsort(fwd)
            rp, ci, va = O.permute_symmetric(a.row_ptr, a.col_idx, a.vals, fwd, inv)
            np.testing.assert_array_equal(rp, golden[f"{name}/{tag}/base_row_ptr"])
            np.testing.assert_array_equal(ci, golden[f"{name}/{tag}/base_col_idx"])
            np.testing.assert_array_equal(va, golden[f"{name}/{tag}/base_vals"])
            for lv in range(k - 1):
                ptr = O.group_pointers(golden[f"{name}/{tag}/sizes{lv}"])
                want = golden[f"{name}/{tag}/ptr{lv}"]
                assert ptr.dtype == want.dtype
                np.testing.assert_array_equal(ptr, want)


def test_oracle_fixture_values():
    # pkg/tests/test_kernels.py:31-46: [[2,0,1,0],[0,3,0,0],[0,0,4,5],[1,0,0,6]] @ [1,2,3,4]
    rp = np.array([0, 2, 3, 5, 7], dtype=np.uint32)
    ci = np.array([0, 2, 1, 2, 3, 0, 3], dtype=np.uint32)
    va = np.array([2.0, 1.0, 3.0, 4.0, 5.0, 1.0, 6.0])
    y = O.spmv_serial(rp, ci, va, np.array([1.0, 2.0, 3.0, 4.0]))
    np.testing.assert_array_equal(y, [5.0, 6.0, 32.0, 25.0])
    # kernels.py:166-175 analogue: 16 ones on 4 lanes -> sum 1..16
    rp = np.array([0, 16], dtype=np.uint32)
    y = O.spmv_strided(rp, np.arange(16, dtype=np.uint32), np.arange(1.0, 17.0),
                       np.ones(16), 4)
    assert y[0] == 136.0


@pytest.mark.parametrize("name", ["grid2d_200", "grid3d7_32", "grid3d27_20",
                                  "grid3d7_24u", "irregular_200k"])
def test_oracle_pipeline_digests(name, configs_golden):
    """Medium configs: native Band-k + oracle pack + oracle CSR-3 reproduce the
    reference's digests (integer arrays and y)."""
    from paper_2203_05096_b200 import CsrMatrix, band_k, csr_from_arrays, synthetic
    rec = configs_golden[name]
    spec = rec["spec"]
    if spec["kind"] == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays(spec["shape"], spec["points"],
                                                 values=spec.get("values", "laplacian"))
        a = CsrMatrix(n, n, rp, ci, va)
    else:
        r, c, v = synthetic.irregular_triplets(spec["rows"], seed=spec.get("seed", 0))
        a = csr_from_arrays(spec["rows"], spec["rows"], r, c, v)
    assert digest(a.row_ptr, "<u4") == rec["input"]["row_ptr"]
    assert digest(a.col_idx, "<u4") == rec["input"]["col_idx"]
    assert digest(a.vals, "<f8") == rec["input"]["vals"]
    x = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
    assert digest(O.spmv_serial(a.row_ptr, a.col_idx, a.vals, x), "<f8") == rec["y_ref"]
    for run in rec["runs"]:
        res = band_k(a, 3, run["targets"])
        assert digest(res.perm.fwd, "<i8") == run["fwd"]
        assert digest(res.level_group_sizes[0], "<i8") == run["sizes0"]
        assert digest(res.level_group_sizes[1], "<i8") == run["sizes1"]
        rp, ci, va = O.permute_symmetric(a.row_ptr, a.col_idx, a.vals, res.perm.fwd,
                                         res.perm.inv)
        assert digest(rp, "<u4") == run["base_row_ptr"]
        assert digest(ci, "<u4") == run["base_col_idx"]
        assert digest(va, "<f8") == run["base_vals"]
        sr = O.group_pointers(res.level_group_sizes[0])
        ssr = O.group_pointers(res.level_group_sizes[1])
        assert digest(sr, "<u4") == run["sr_ptr"]
        assert digest(ssr, "<u4") == run["ssr_ptr"]
        xp = O.gather(x, res.perm.inv)
        assert digest(xp, "<f8") == run["xp"]
        y3 = O.spmv_grouped(O.csr3_group_rows(sr, ssr), rp, ci, va, xp, workers=4)
        assert digest(y3, "<f8") == run["y_csr3"]
        if "y_emu35_4x8x12" in run:
            assert digest(O.spmv_strided(rp, ci, va, xp, 4), "<f8") == run["y_emu35_4x8x12"]
