"""Full-size configurations (BASELINE.json configs C2, C3, C5) against the
digests the unmodified reference produced (tests/golden/configs.json, ~5 min
of reference Band-k each): device and host Band-k permutations and group
sizes, the device-packed CSR-k arrays, y of the CSR-3 kernel and y of the
strided (GPUSpMV-3.5) order -- at the Volta model's targets and at the
B200 model's targets, i.e. exactly the matrix and order bench.py times."""

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
    # the bench's matrix: the B200 model's targets must be one of the runs
    params = ck.tune_gpu(ck.compute_stats(a), ck.b200_profile())
    assert [params.srs, params.ssrs] in [r["targets"] for r in rec["runs"]]
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
        for key in [k for k in run if k.startswith("y_emu35_")]:
            dims = ck.BlockDims(*(int(v) for v in key[len("y_emu35_"):].split("x")))
            assert digest(ck.spmv_gpu35(m, xp, dims), "<f8") == run[key], key
        with capsys.disabled():
            print(f"\n[{name}] device band_k {t_dev:.2f}s (reference {run['band_k_seconds']}s)")
    if name == "C2":  # the host implementation too, once
        t0 = time.perf_counter()
        res = ck.band_k(a, 3, rec["runs"][0]["targets"], backend="host")
        t_host = time.perf_counter() - t0
        assert digest(res.perm.fwd, "<i8") == rec["runs"][0]["fwd"]
        with capsys.disabled():
            print(f"[{name}] host band_k {t_host:.2f}s")


_OFFS7 = ((-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0))


def _stencil7_cols(i, n):
    """Columns of row i of the n^3 7-point Laplacian, ascending."""
    z, y, x = i // (n * n), (i // n) % n, i % n
    out = []
    for dz, dy, dx in _OFFS7:
        zz, yy, xx = z + dz, y + dy, x + dx
        if 0 <= zz < n and 0 <= yy < n and 0 <= xx < n:
            out.append((zz * n + yy) * n + xx)
    return out


@pytest.mark.parametrize("variant", ["serial", "strided"])
def test_c4_full_size_properties(variant):
    """C4 (512^3, 938 M nonzeros) where no CPU oracle fits:
    x = 1 gives y_i = 6 - (in-grid neighbours of i) exactly, and 20,000
    sampled rows of a random x equal the reference's row order bit for bit
    (serial order; the strided order is checked on the x = 1 property)."""
    torch = pytest.importorskip("torch")
    n = 512
    dev = synthetic.device_stencil((n, n, n), 7).group_uniform(8, 8)
    assert dev.nnz == 7 * n ** 3 - 6 * n ** 2
    rows = n ** 3
    dims = ck.BlockDims(4, 8, 8)
    ones = torch.ones(rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(ones)
    ck.spmv_device(dev, ones, y, dims=dims, variant=variant)
    idx = torch.arange(rows, device="cuda", dtype=torch.int64)
    xi, yi, zi = idx % n, (idx // n) % n, idx // (n * n)
    deg = torch.zeros_like(idx)
    for c in (xi, yi, zi):
        deg += (c > 0).long() + (c < n - 1).long()
    assert torch.equal(y, (6 - deg).double())
    del idx, xi, yi, zi, deg
    if variant != "serial":
        return
    g = torch.Generator(device="cuda").manual_seed(3)
    xr = torch.rand(rows, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    ck.spmv_device(dev, xr, y, variant="serial")
    rng = np.random.default_rng(4)
    sample = np.concatenate([rng.integers(0, rows, 20000), [0, rows - 1, n * n - 1, n - 1]])
    ys = y[torch.from_numpy(sample).cuda()].cpu().numpy()
    cols = [_stencil7_cols(int(i), n) for i in sample]
    flat = np.array([c for cs in cols for c in cs], dtype=np.int64)
    xv = xr[torch.from_numpy(flat).cuda()].cpu().numpy()
    pos = 0
    for k, i in enumerate(sample.tolist()):
        acc = 0.0  # the reference's left-to-right row sum (kernels.py:117-147)
        for j in cols[k]:
            acc += (6.0 if j == i else -1.0) * float(xv[pos])
            pos += 1
        assert ys[k] == acc, i
