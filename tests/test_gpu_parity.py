"""GPU parity: the sm_100a kernels against the reference's golden outputs and
the CPU oracle.  Integer arrays and fp64 y are compared bit for bit
(SURVEY.md §8(c)); fp32 within 1e-5 of the |A||x| scale."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from conftest import BANDK_TAGS, digest, random_csr
from oracle import oracle as O
from paper_2203_05096_b200 import _native, synthetic
from paper_2203_05096_b200.kernels import STRIDED_NX

pytestmark = pytest.mark.gpu

EMU35_DIMS = [(4, 8, 12), (8, 8, 8), (16, 8, 4), (2, 2, 2), (3, 5, 2), (1, 3, 4), (32, 2, 2)]
EMU3_DIMS = [(8, 12, 1), (1, 1, 1), (5, 3, 1)]


def _trace_array(tr):
    return np.stack([tr.row, tr.block, tr.z_lane, tr.y_lane, tr.x_first, tr.x_count,
                     tr.reduction_depth])


def test_plain_csr_kernel_bitwise(golden):
    for name in golden.names:
        a = golden.csr(name)
        for xs in ("pos", "sgn"):
            y = ck.spmv_csr_ref(a, golden[f"{name}/x_{xs}"])
            np.testing.assert_array_equal(y, golden[f"{name}/y_ref_{xs}"], err_msg=name)


def test_device_pack_and_kernels_bitwise(golden):
    for name in golden.names:
        a = golden.csr(name)
        for tag, k, _ in BANDK_TAGS:
            p = f"{name}/{tag}"
            fwd = golden[f"{p}/fwd"]
            perm = ck.Permutation.from_forward(fwd)
            sizes = [golden[f"{p}/sizes{lv}"].tolist() for lv in range(k - 1)]
            m = ck.pack_csrk(a, perm, sizes)
            np.testing.assert_array_equal(m.base.row_ptr, golden[f"{p}/base_row_ptr"])
            np.testing.assert_array_equal(m.base.col_idx, golden[f"{p}/base_col_idx"])
            np.testing.assert_array_equal(m.base.vals, golden[f"{p}/base_vals"])
            for lv in range(k - 1):
                assert m.group_ptrs[lv].dtype == np.uint32
                np.testing.assert_array_equal(m.group_ptrs[lv], golden[f"{p}/ptr{lv}"])
            for xs in ("pos", "sgn"):
                x = golden[f"{name}/x_{xs}"]
                xp = ck.permute_vector(perm, x)
                np.testing.assert_array_equal(xp, x[perm.inv])
                np.testing.assert_array_equal(ck.unpermute_vector(perm, xp), x)
                if k == 2:
                    np.testing.assert_array_equal(ck.spmv_csr2(m, xp),
                                                  golden[f"{p}/y_csr2_{xs}"])
                    continue
                y3 = golden[f"{p}/y_csr3_{xs}"]
                np.testing.assert_array_equal(ck.spmv_csr3(m, xp), y3, err_msg=f"{p}")
                for d in EMU3_DIMS:
                    y, tr = ck.emulate_gpu_spmv3(m, xp, ck.BlockDims(*d))
                    np.testing.assert_array_equal(y, y3)
                    tr.validate_partition(a.n_rows)
                    key = f"{p}/trace_emu3_{'x'.join(map(str, d))}"
                    if xs == "pos" and golden.has(key):
                        np.testing.assert_array_equal(_trace_array(tr), golden[key])
                for d in EMU35_DIMS:
                    dt = "x".join(map(str, d))
                    key = f"{p}/y_emu35_{dt}_{xs}"
                    y, tr = ck.emulate_gpu_spmv35(m, xp, ck.BlockDims(*d))
                    if golden.has(key):
                        np.testing.assert_array_equal(y, golden[key], err_msg=f"{p} {d}")
                    else:
                        np.testing.assert_array_equal(
                            y, O.spmv_strided(m.base.row_ptr, m.base.col_idx, m.base.vals,
                                              xp, d[0]))
                    tkey = f"{p}/trace_emu35_{dt}"
                    if xs == "pos" and golden.has(tkey):
                        np.testing.assert_array_equal(_trace_array(tr), golden[tkey])
                    if d[0] in STRIDED_NX:
                        np.testing.assert_array_equal(ck.spmv_gpu35(m, xp, ck.BlockDims(*d)),
                                                      y, err_msg=f"stream {p} {d}")


def test_device_stats_bitwise(golden):
    for name in golden.names:
        a = golden.csr(name)
        s = ck.compute_stats(a)
        want = golden[f"{name}/stats"]
        assert s.rdensity == want[0]
        assert s.variance == want[1], name
        assert s.pattern_symmetry == want[2]
        assert s.max_row_nnz == int(want[3])


def test_stats_reference_cases():
    counts = [10, 10, 0, 0, 5, 5, 5, 5, 5, 5]
    a = ck.build_csr(10, 10, [(i, j, 1.0) for i, c in enumerate(counts) for j in range(c)])
    s = ck.compute_stats(a)
    assert s.variance == 10.0 and ck.classify(s) is ck.MatrixClass.REGULAR
    upper = ck.build_csr(3, 3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)])
    assert ck.compute_stats(upper).pattern_symmetry == 0.0
    diag = ck.build_csr(3, 3, [(i, i, 1.0) for i in range(3)])
    assert ck.compute_stats(diag).pattern_symmetry == 1.0
    rng = np.random.default_rng(5)
    big = random_csr(rng, 3000, 3000, 0.004)
    counts = np.diff(big.row_ptr.astype(np.int64))
    assert ck.compute_stats(big).variance == float(np.var(counts))


def test_edge_cases():
    # empty and zero matrices (pkg/tests/test_kernels.py:49-57)
    assert ck.spmv_csr_ref(ck.build_csr(0, 0, []), np.zeros(0)).shape == (0,)
    np.testing.assert_array_equal(ck.spmv_csr_ref(ck.build_csr(3, 4, []), np.ones(4)),
                                  np.zeros(3))
    x = np.linspace(-2, 2, 5)
    np.testing.assert_array_equal(
        ck.spmv_csr_ref(ck.build_csr(5, 5, [(i, i, 1.0) for i in range(5)]), x), x)
    # one group holding every row; one super-row per row
    rng = np.random.default_rng(11)
    a = random_csr(rng, 30, 30, 0.2, -1.0, 1.0)
    x = rng.uniform(-1.0, 1.0, 30)
    ref = O.spmv_serial(a.row_ptr, a.col_idx, a.vals, x)
    p = ck.Permutation.identity(30)
    np.testing.assert_array_equal(ck.spmv_csr2(ck.pack_csrk(a, p, [[30]]), x), ref)
    np.testing.assert_array_equal(ck.spmv_csr3(ck.pack_csrk(a, p, [[30], [1]]), x), ref)
    np.testing.assert_array_equal(ck.spmv_csr3(ck.pack_csrk(a, p, [[1] * 30, [30]]), x), ref)


def _long_row_matrix(rng, n, long_len, n_long=2):
    rows, cols = [], []
    for r in range(n):
        k = long_len if r % max(1, n // n_long) == 0 else int(rng.integers(0, 12))
        c = np.sort(rng.choice(n, size=min(k, n), replace=False))
        rows.append(np.full(len(c), r))
        cols.append(c)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    return ck.csr_from_arrays(n, n, rows, cols, rng.uniform(-1.0, 1.0, len(rows)))


@pytest.mark.parametrize("long_len", [33, 129, 300, 5000, 40000])
def test_long_rows_pack_and_spmv(long_len):
    """Rows longer than a warp / the shared stage: the device pack sorts them
    (bitonic paths) and the streaming kernel's long-row path keeps the
    reference's order."""
    rng = np.random.default_rng(long_len)
    n = 60000
    a = _long_row_matrix(rng, n, long_len)
    fwd = rng.permutation(n)
    perm = ck.Permutation.from_forward(fwd)
    sizes1 = [4] * (n // 4)
    sizes2 = [5] * (len(sizes1) // 5)
    m = ck.pack_csrk(a, perm, [sizes1, sizes2])
    rp, ci, va = O.permute_symmetric(a.row_ptr, a.col_idx, a.vals, perm.fwd, perm.inv)
    np.testing.assert_array_equal(m.base.row_ptr, rp)
    np.testing.assert_array_equal(m.base.col_idx, ci)
    np.testing.assert_array_equal(m.base.vals, va)
    x = rng.uniform(-1.0, 1.0, n)
    np.testing.assert_array_equal(ck.spmv_csr3(m, x), O.spmv_serial(rp, ci, va, x))
    for nx in (1, 3, 4, 8, 12, 32):
        np.testing.assert_array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(nx, 1, 1)),
                                      O.spmv_strided(rp, ci, va, x, nx), err_msg=str(nx))


@pytest.mark.parametrize("tile_cost,cap,stages", [(16, 16, 1), (64, 40, 2), (4096, 4400, 2),
                                                  (300, 17, 4), (1000, 0, 8), (0, 0, 0)])
def test_tile_plans_do_not_change_bits(tile_cost, cap, stages):
    rng = np.random.default_rng(tile_cost + cap + stages)
    n = 20000
    a = random_csr(rng, n, n, 6.0 / n, -1.0, 1.0)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = rng.uniform(-1.0, 1.0, n)
    want = O.spmv_grouped(O.csr3_group_rows(m.sr_ptr, m.ssr_ptr), m.base.row_ptr,
                          m.base.col_idx, m.base.vals, x, 1)
    m.device().set_plan(tile_cost, cap, stages)
    np.testing.assert_array_equal(ck.spmv_csr3(m, x), want)
    np.testing.assert_array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(4, 8, 12)),
                                  O.spmv_strided(m.base.row_ptr, m.base.col_idx,
                                                 m.base.vals, x, 4))


def test_device_resident_and_fp32():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(2)
    n, rp, ci, va = synthetic.stencil_arrays((40, 40, 40), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = rng.uniform(-1.0, 1.0, n)
    want = ck.spmv_csr3(m, x)
    xd = torch.from_numpy(x).cuda()
    yd = ck.spmv_device(m, xd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(yd.cpu().numpy(), want)
    y32 = ck.spmv_device(m, xd.float())
    torch.cuda.synchronize()
    scale = O.abs_row_dot(m.base.row_ptr, m.base.col_idx, m.base.vals, x)
    err = np.abs(y32.cpu().double().numpy() - want) / scale
    assert err.max() <= 1e-5  # north_star fp32 tolerance
    y32s = ck.spmv_device(m, xd.float(), dims=ck.BlockDims(4, 8, 12), variant="strided")
    torch.cuda.synchronize()
    assert (np.abs(y32s.cpu().double().numpy() - want) / scale).max() <= 1e-5


@pytest.mark.parametrize("shape,points", [((37, 41), 5), ((23, 19), 9), ((11, 13, 17), 7),
                                          ((9, 10, 11), 27)])
def test_device_stencil_generator_matches_host(shape, points):
    dev = synthetic.device_stencil(shape, points)
    rp, ci, va, _, _ = dev.download()
    n, hrp, hci, hva = synthetic.stencil_arrays(shape if len(shape) == 3 else shape, points)
    np.testing.assert_array_equal(rp, hrp)
    np.testing.assert_array_equal(ci, hci)
    np.testing.assert_array_equal(va, hva)


@pytest.mark.parametrize("name", ["grid2d_200", "grid3d7_32", "grid3d27_20", "grid3d7_24u",
                                  "irregular_200k", "C1"])
def test_pipeline_digests_vs_reference(name, configs_golden):
    """Full drop-in pipeline at medium size: Band-k -> device pack -> CSR-3
    kernel and the Listing-4 / strided kernels, digests equal to the
    reference's."""
    rec = configs_golden[name]
    spec = rec["spec"]
    if spec["kind"] == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays(spec["shape"], spec["points"],
                                                 values=spec.get("values", "laplacian"))
        a = ck.CsrMatrix(n, n, rp, ci, va)
    else:
        r, c, v = synthetic.irregular_triplets(spec["rows"], seed=spec.get("seed", 0))
        a = ck.csr_from_arrays(spec["rows"], spec["rows"], r, c, v)
    x = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
    assert digest(ck.spmv_csr_ref(a, x), "<f8") == rec["y_ref"]
    st = ck.compute_stats(a)
    assert float(st.variance).hex() == rec["stats"]["variance"]
    assert float(st.pattern_symmetry).hex() == rec["stats"]["pattern_symmetry"]
    assert ck.tune_gpu(st, ck.VOLTA).to_dict() == rec["tune_volta"]
    for run in rec["runs"]:
        res = ck.band_k(a, 3, run["targets"])
        assert digest(res.perm.fwd, "<i8") == run["fwd"]
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
        if "y_emu35_4x8x12" in run:
            dims = ck.BlockDims(4, 8, 12)
            assert digest(ck.emulate_gpu_spmv35(m, xp, dims)[0], "<f8") == run["y_emu35_4x8x12"]
            assert digest(ck.spmv_gpu35(m, xp, dims), "<f8") == run["y_emu35_4x8x12"]


def test_native_library_is_loaded():
    import paper_2203_05096_b200._native as nat
    assert nat._lib is not None or nat.lib() is not None
    assert nat.device_count() >= 1


def test_pinned_host_pipeline_bitwise():
    """Pinned host buffers take the chunked, overlapped H2D / kernel / D2H
    pipeline; results equal the plain path and the oracle bit for bit."""
    torch = pytest.importorskip("torch")
    n, rp, ci, va = synthetic.stencil_arrays((96, 112, 128), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = np.random.default_rng(4).uniform(-1.0, 1.0, n)
    plain = ck.spmv_csr3(m, x)
    want = O.spmv_grouped(O.csr3_group_rows(m.sr_ptr, m.ssr_ptr), m.base.row_ptr,
                          m.base.col_idx, m.base.vals, x, 4)
    np.testing.assert_array_equal(plain, want)
    x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    x_pin[:] = x
    for _ in range(3):
        y_pin[:] = np.nan
        ck.spmv_csr3(m, x_pin, out=y_pin)
        np.testing.assert_array_equal(y_pin, want)
    m.device().spmv_host(x_pin, variant=_native.CSRK_STRIDED, nx=4, out=y_pin)
    np.testing.assert_array_equal(
        y_pin, O.spmv_strided(m.base.row_ptr, m.base.col_idx, m.base.vals, x, 4))


def test_plan_geometry_checks():
    rng = np.random.default_rng(1)
    a = random_csr(rng, 500, 500, 0.01)
    dev = a.device()
    with pytest.raises(ValueError, match="shared memory"):
        dev.set_plan(65536, 70000, 8)
    dev.set_plan(512, 0, 2)
    plan = dev.plan()
    assert plan["tile_cost"] == 512 and plan["stages"] == 2
    assert plan["n_tiles"] == -(-(a.nnz + a.n_rows) // 512)


def _mixed_rows_matrix(rng, n):
    """Rows of 0..60 nonzeros (mean > 16, variance >> 10) plus long rows of
    129..1500 nonzeros (holes inside staged tiles) and 3000: exercises every
    schedule's inline, gather-first, direct and long-row paths."""
    lens = rng.integers(0, 61, n)
    lens[rng.choice(n, 60, replace=False)] = rng.integers(129, 1500, 60)
    lens[rng.choice(n, 5, replace=False)] = 3000
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, len(rows))
    return ck.csr_from_arrays(n, n, rows, cols, rng.uniform(-1.0, 1.0, len(rows)))


@pytest.mark.parametrize("tile_cost,stages", [(0, 0), (256, 3), (1153, 2), (4096, 2)])
def test_long_row_tile_cuts(tile_cost, stages):
    """With long rows present the plan has no empty tiles, and a tile whose
    nonzeros exceed its stage is one (long) row -- the cuts around long rows
    (spmv.cu recut_long) -- while both orders keep the oracle's bits."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(tile_cost + stages)
    n = 40000
    lens = rng.integers(0, 20, n)
    lens[rng.choice(n, 300, replace=False)] = rng.integers(129, 6000, 300)
    rows = np.repeat(np.arange(n), lens)
    a = ck.csr_from_arrays(n, n, rows, rng.integers(0, n, len(rows)),
                           rng.uniform(-1.0, 1.0, len(rows)))
    m = ck.pack_csrk(a, ck.Permutation.identity(n), [[1] * n, [n]])
    dev = m.device()
    dev.set_plan(tile_cost, 0, stages)
    plan = dev.plan()
    tr = dev.tile_rows().astype(np.int64)
    assert tr[0] == 0 and tr[-1] == n and len(tr) == plan["n_tiles"] + 1
    assert np.all(np.diff(tr) > 0)
    rp = a.row_ptr.astype(np.int64)
    big = rp[tr[1:]] - rp[tr[:-1]] > plan["cap"]
    assert np.all(np.diff(tr)[big] == 1)
    x = rng.uniform(-1.0, 1.0, n)
    np.testing.assert_array_equal(ck.spmv_csr3(m, x), O.spmv_serial(a.row_ptr, a.col_idx,
                                                                    a.vals, x))
    for nx in (4, 8):
        np.testing.assert_array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(nx, 1, 1)),
                                      O.spmv_strided(a.row_ptr, a.col_idx, a.vals, x, nx))
    # fp32 (16-byte segments of 4 values around the holes), odd lane counts
    want = O.spmv_serial(a.row_ptr, a.col_idx, a.vals, x)
    scale = O.abs_row_dot(a.row_ptr, a.col_idx, a.vals, x)
    xd = torch.from_numpy(x).cuda().float()
    for variant, nx in (("serial", 1), ("strided", 3), ("strided", 12)):
        y32 = ck.spmv_device(m, xd, dims=ck.BlockDims(nx, 1, 1), variant=variant)
        torch.cuda.synchronize()
        assert np.all(np.abs(y32.cpu().double().numpy() - want) <= 1e-5 * scale)  # empty rows: 0


@pytest.mark.parametrize("gather,ctas", [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 3),
                                         (0, 4), (1, 8), (2, 2)])
def test_schedules_do_not_change_bits(gather, ctas):
    """Gather mode x CTAs/SM x tile plan: y is the oracle's bit for bit in
    both orders (f64) and within 1e-5 of |A||x| (f32)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(10 * gather + ctas)
    n = 30000
    a = _mixed_rows_matrix(rng, n)
    res = ck.band_k(a, 3, [4, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = rng.uniform(-1.0, 1.0, n)
    rp, ci, va = m.base.row_ptr, m.base.col_idx, m.base.vals
    want = O.spmv_serial(rp, ci, va, x)
    want4 = O.spmv_strided(rp, ci, va, x, 4)
    scale = O.abs_row_dot(rp, ci, va, x)
    dev = m.device()
    dev.set_schedule(gather, ctas)
    for tile_cost, stages in ((0, 0), (256, 3), (4096, 2), (700, 1)):
        dev.set_plan(tile_cost, 0, stages)
        plan = dev.plan()
        assert plan["gather_first"] == gather
        assert plan["ctas_per_sm"] == (ctas or 2)  # variance >> 10: irregular
        np.testing.assert_array_equal(ck.spmv_csr3(m, x), want)
        np.testing.assert_array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(4, 8, 12)), want4)
        xd = torch.from_numpy(x).cuda().float()
        y32 = ck.spmv_device(m, xd)
        torch.cuda.synchronize()
        assert (np.abs(y32.cpu().double().numpy() - want) / np.maximum(scale, 1e-300)).max() <= 1e-5


def test_schedule_argument_checks():
    rng = np.random.default_rng(3)
    dev = random_csr(rng, 300, 300, 0.02).device()
    with pytest.raises(ValueError, match="gather"):
        dev.set_schedule(3, 0)
    with pytest.raises(ValueError, match="ctas_per_sm"):
        dev.set_schedule(0, 9)


@pytest.mark.parametrize("shape,d2h,xcut", [("u1", "host", "footprint"), ("u3", "event", "rows"),
                                            ("r1", "host", "rows"), ("r12", "event", "footprint"),
                                            ("u40", "host", "footprint")])
def test_pipeline_shapes_bitwise(monkeypatch, shape, d2h, xcut):
    """Every host-pipeline chunking / ordering gives the plain path's bits."""
    torch = pytest.importorskip("torch")
    n, rp, ci, va = synthetic.stencil_arrays((64, 128, 160), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    want = O.spmv_grouped(O.csr3_group_rows(m.sr_ptr, m.ssr_ptr), m.base.row_ptr,
                          m.base.col_idx, m.base.vals, x, 4)
    monkeypatch.setenv("CSRK_PIPE_SHAPE", shape)
    monkeypatch.setenv("CSRK_PIPE_D2H", d2h)
    monkeypatch.setenv("CSRK_PIPE_XCUT", xcut)
    x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    x_pin[:] = x
    for _ in range(2):
        y_pin[:] = np.nan
        ck.spmv_csr3(m, x_pin, out=y_pin)
        np.testing.assert_array_equal(y_pin, want)


@pytest.mark.parametrize("shape", ["u3", "r12"])
def test_pipeline_with_long_rows(monkeypatch, shape):
    """The pinned host pipeline's chunked tile-range launches with long rows
    (each chunk's long rows, the side stream for nx = 4): the oracle's bits."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    n = 1_200_000  # > 1 M rows: the pinned pipeline engages
    lens = rng.integers(0, 12, n)
    lens[rng.choice(n, 500, replace=False)] = rng.integers(129, 3000, 500)
    rows = np.repeat(np.arange(n), lens)
    a = ck.csr_from_arrays(n, n, rows, np.minimum(n - 1, rows + rng.integers(0, 5000, len(rows))),
                           rng.uniform(-1.0, 1.0, len(rows)))
    m = ck.pack_csrk(a, ck.Permutation.identity(n), [[1] * n, [n]])
    monkeypatch.setenv("CSRK_PIPE_SHAPE", shape)
    x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    x_pin[:] = rng.uniform(-1.0, 1.0, n)
    y_pin[:] = np.nan
    ck.spmv_csr3(m, x_pin, out=y_pin)
    np.testing.assert_array_equal(y_pin, O.spmv_serial(a.row_ptr, a.col_idx, a.vals, x_pin))
    y_pin[:] = np.nan
    ck.spmv_gpu35(m, x_pin, ck.BlockDims(4, 1, 1), out=y_pin)
    np.testing.assert_array_equal(y_pin, O.spmv_strided(a.row_ptr, a.col_idx, a.vals, x_pin, 4))


def test_auto_plan_follows_the_order():
    """An automatic plan (tile 1536, a 3-stage ring for regular rows)
    re-tiles strided launches only when their rows would leave a pass mostly
    empty, keeps 1536 for the serial order, and never changes bits --
    including the pinned host pipeline run right after a re-plan."""
    torch = pytest.importorskip("torch")
    n, rp, ci, va = synthetic.stencil_arrays((100, 100, 105), 27, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)  # > 1 M rows: the pinned pipeline engages
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = np.random.default_rng(9).uniform(-1.0, 1.0, n)
    b = m.base
    want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)
    dev = m.device()
    for _ in range(2):
        np.testing.assert_array_equal(ck.spmv_csr3(m, x), want)
        assert dev.plan()["tile_cost"] == 1536 and dev.plan()["stages"] == 3
        for nx in (2, 4, 8, 32):
            np.testing.assert_array_equal(ck.spmv_gpu35(m, x, ck.BlockDims(nx, 1, 1)),
                                          O.spmv_strided(b.row_ptr, b.col_idx, b.vals, x, nx))
            tc = dev.plan()["tile_cost"]
            assert (512 <= tc <= 1536) and dev.plan()["stages"] == 3
    x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    x_pin[:] = x
    ck.spmv_gpu35(m, x_pin, ck.BlockDims(4, 1, 1), out=y_pin)
    np.testing.assert_array_equal(y_pin, O.spmv_strided(b.row_ptr, b.col_idx, b.vals, x, 4))
    ck.spmv_csr3(m, x_pin, out=y_pin)
    np.testing.assert_array_equal(y_pin, want)
    dev.set_plan(1000, 0, 2)  # explicit plans stay put
    ck.spmv_gpu35(m, x, ck.BlockDims(4, 1, 1))
    assert dev.plan()["tile_cost"] == 1000


@pytest.mark.parametrize("cut_mode", [0, 1, 2])
@pytest.mark.parametrize("kind", ["mixed", "stencil", "irregular", "empty_rows"])
def test_cut_modes_bitwise(cut_mode, kind):
    """Tile cuts on rows, on super-super-row boundaries (the paper's SSR ->
    block mapping) or auto give the reference's row order bit for bit, under
    several plans (staged and direct tiles), for whole launches and tile
    ranges; group cuts fall only on SSR starts."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(len(kind) + cut_mode)
    if kind == "mixed":
        a = _mixed_rows_matrix(rng, 20000)
    elif kind == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays((30, 31, 32), 7, values="uniform")
        a = ck.CsrMatrix(n, n, rp, ci, va)
    elif kind == "irregular":
        r, c, v = synthetic.irregular_triplets(60000, seed=3)
        a = ck.csr_from_arrays(60000, 60000, r, c, v)
    else:  # every third row empty, others 1..40 nonzeros
        n = 30000
        lens = rng.integers(1, 41, n)
        lens[::3] = 0
        rows = np.repeat(np.arange(n), lens)
        a = ck.csr_from_arrays(n, n, rows, rng.integers(0, n, len(rows)),
                               rng.uniform(-1, 1, len(rows)))
    res = ck.band_k(a, 3, [4, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    b = m.base
    x = rng.uniform(-1.0, 1.0, b.n_rows)
    want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)
    dev = m.device()
    dev.set_cut_mode(cut_mode)
    xd = torch.from_numpy(x).cuda()
    ssr_rows = set((m.sr_ptr.astype(np.int64)[m.ssr_ptr.astype(np.int64)]).tolist())
    for tile_cost, stages in ((0, 0), (256, 3), (4096, 2), (48, 1)):
        dev.set_plan(tile_cost, 0, stages)
        np.testing.assert_array_equal(ck.spmv_csr3(m, x), want)
        plan = dev.plan()
        assert plan["cut_mode"] == cut_mode
        if cut_mode == 2 and plan["n_long"] == 0:
            assert plan["group_aligned"] == 1
            assert set(dev.tile_rows().tolist()) <= ssr_rows
            # groups larger than the tile: the pitch stays >= a tile (it
            # used to drop to 1 and multiply the tile count by the tile cost)
            assert plan["n_tiles"] <= 4 * (b.nnz + b.n_rows) // plan["tile_cost"] + 8
        yd = torch.full_like(xd, float("nan"))
        nt = plan["n_tiles"]
        cut = nt // 3
        for t0, t1 in ((0, cut), (cut, nt)):
            dev.spmv_tiles_ptr(xd.data_ptr(), yd.data_ptr(), t0, t1,
                               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(yd.cpu().numpy(), want)


def test_tile_range_and_cut_mode_argument_checks():
    """The C-ABI rejects bad tile ranges and cut modes with ValueError."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    a = random_csr(rng, 2000, 2000, 0.004)
    dev = a.device()
    dev.set_plan(64, 0, 2)
    nt = dev.plan()["n_tiles"]
    x = torch.zeros(2000, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    s = torch.cuda.current_stream().cuda_stream
    with pytest.raises(ValueError, match="tile range"):
        dev.spmv_tiles_ptr(x.data_ptr(), y.data_ptr(), 0, nt + 1, s)
    with pytest.raises(ValueError, match="tile range"):
        dev.spmv_tiles_ptr(x.data_ptr(), y.data_ptr(), 3, 2, s)
    dev.spmv_tiles_ptr(x.data_ptr(), y.data_ptr(), 2, 2, s)  # empty range: no-op
    with pytest.raises(ValueError, match="cut mode"):
        dev.set_cut_mode(3)
    tr = dev.tile_rows()
    assert tr[0] == 0 and tr[-1] == 2000 and len(tr) == nt + 1 and np.all(np.diff(tr) >= 0)
