"""CG / repeated-SpMV loops around the CSR-k kernel:
agreement with a float64 numpy CG, determinism, CUDA-graph replay, and the
device stencil + uniform grouping path used for C4."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from oracle import oracle as O
from paper_2203_05096_b200 import cg, synthetic

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _numpy_cg(rp, ci, va, b, iters):
    def matvec(v):
        return O.spmv_serial(rp, ci, va, v)
    x = np.zeros_like(b)
    r = b - matvec(x)
    p = r.copy()
    rr = r @ r
    for _ in range(iters):
        ap = matvec(p)
        alpha = rr / (p @ ap)
        x += alpha * p
        r -= alpha * ap
        rr_new = r @ r
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, rr


def _laplacian(shape=(24, 24, 24)):
    n, rp, ci, va = synthetic.stencil_arrays(shape, 7)
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    return a, res, ck.pack_csrk(a, res.perm, res.level_group_sizes)


def test_cg_matches_numpy_and_converges():
    a, res, m = _laplacian()
    n = a.n_rows
    b_np = np.random.default_rng(0).uniform(-1, 1, n)[res.perm.inv]
    x_ref, rr_ref = _numpy_cg(m.base.row_ptr, m.base.col_idx, m.base.vals, b_np, 60)
    b = torch.from_numpy(b_np).cuda()
    x, info = cg.cg(m, b, iters=60)
    xs = x.cpu().numpy()
    assert np.abs(xs - x_ref).max() <= 1e-9 * np.abs(x_ref).max()
    assert info["rr"] == pytest.approx(rr_ref, rel=1e-6)
    resid = b_np - O.spmv_serial(m.base.row_ptr, m.base.col_idx, m.base.vals, xs)
    assert np.linalg.norm(resid) < 1e-3 * np.linalg.norm(b_np)
    # deterministic: a second run gives the same bits
    x2, _ = cg.cg(m, b, iters=60)
    assert torch.equal(x, x2)


def test_cg_graph_replay_equals_eager_and_fp32():
    a, res, m = _laplacian((20, 20, 20))
    n = a.n_rows
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    x_eager, _ = cg.cg(m, b, iters=25)
    x = torch.zeros_like(b)
    scratch = tuple(torch.empty_like(b) for _ in range(3))

    def loop(stream):
        x.zero_()
        cg.cg(m, b, x, iters=25, stream=stream, scratch=scratch, sync=False)

    g = cg.GraphedLoop(loop)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, x_eager)
    x32, info32 = cg.cg(m, b.float(), iters=25)
    assert (x32.double() - x_eager).abs().max().item() < 1e-3 * x_eager.abs().max().item()


def test_power_iterations_normalise():
    a, res, m = _laplacian((16, 16, 16))
    n = a.n_rows
    x0 = np.random.default_rng(2).uniform(0.5, 1.5, n)
    x = torch.from_numpy(x0.copy()).cuda()
    cg.power_iterations(m, x, iters=5)
    v = x0.copy()
    for _ in range(5):
        yv = O.spmv_serial(m.base.row_ptr, m.base.col_idx, m.base.vals, v)
        v = yv * (1.0 / np.abs(yv).max())
    np.testing.assert_array_equal(x.cpu().numpy(), v)


def test_device_stencil_uniform_groups():
    dev = synthetic.device_stencil((30, 31, 32), 7).group_uniform(8, 8)
    assert dev.k == 3 and dev.n_sr == -(-dev.n_rows // 8)
    rp, ci, va, sp, ssp = dev.download()
    assert sp[-1] == dev.n_rows and ssp[-1] == dev.n_sr
    x = np.random.default_rng(3).uniform(-1, 1, dev.n_rows)
    np.testing.assert_array_equal(dev.spmv_host(x), O.spmv_serial(rp, ci, va, x))
    # the C4 analytic check: Laplacian row sums are 7 - row length
    y1 = dev.spmv_host(np.ones(dev.n_rows))
    np.testing.assert_array_equal(y1, 7.0 - np.diff(rp.astype(np.int64)))


def _arrowhead(n=6000, hubs=(0, 1500, 4000), step=3):
    """SPD, diagonally dominant, with dense hub rows / columns: rows longer
    than 128 nonzeros go to the long-row kernel (and, strided nx <= 8, its
    side stream) inside the CG / power loops."""
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.full(n, 10.0)]
    for h in hubs:
        c = np.arange(0, n, step)
        c = c[c != h]
        rows += [np.full(len(c), h), c]
        cols += [c, np.full(len(c), h)]
        vals += [np.full(len(c), 1e-3), np.full(len(c), 1e-3)]
    a = ck.csr_from_arrays(n, n, np.concatenate(rows), np.concatenate(cols),
                           np.concatenate(vals))
    res = ck.band_k(a, 3, [4, 8])
    return a, res, ck.pack_csrk(a, res.perm, res.level_group_sizes)


@pytest.mark.parametrize("variant,nx", [("serial", 0), ("strided", 4), ("strided", 16)])
def test_long_rows_in_cg_graph_and_power(variant, nx):
    a, res, m = _arrowhead()
    rp, ci, va = m.base.row_ptr, m.base.col_idx, m.base.vals
    assert np.diff(rp).max() > 128
    n = a.n_rows
    dims = ck.BlockDims(max(nx, 1), 1, 1)
    b = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, n)).cuda()
    x_eager, info = cg.cg(m, b, iters=30, dims=dims, variant=variant)
    x = torch.zeros_like(b)
    scratch = tuple(torch.empty_like(b) for _ in range(3))

    def loop(stream):
        x.zero_()
        cg.cg(m, b, x, iters=30, dims=dims, variant=variant, stream=stream,
              scratch=scratch, sync=False)

    g = cg.GraphedLoop(loop)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, x_eager)
    resid = b.cpu().numpy() - O.spmv_serial(rp, ci, va, x.cpu().numpy())
    assert np.linalg.norm(resid) < 1e-8 * np.linalg.norm(b.cpu().numpy())
    # power iterations: bit for bit the oracle's order
    x0 = np.random.default_rng(5).uniform(0.5, 1.5, n)
    xp = torch.from_numpy(x0.copy()).cuda()
    cg.power_iterations(m, xp, iters=4, dims=dims, variant=variant)
    v = x0.copy()
    for _ in range(4):
        yv = (O.spmv_serial(rp, ci, va, v) if variant == "serial"
              else O.spmv_strided(rp, ci, va, v, nx))
        v = yv * (1.0 / np.abs(yv).max())
    np.testing.assert_array_equal(xp.cpu().numpy(), v)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_cg_fused_dot_matches_separate_dot(dtype, monkeypatch):
    """p . Ap fused into the SpMV epilogue (per-CTA partials, fixed order)
    against the separate dot kernel (CSRK_NO_FUSED_DOT=1): same iterates up
    to the reduction order, deterministic run to run."""
    a, res, m = _laplacian((28, 28, 28))
    n = a.n_rows
    b = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, n)).cuda()
    if dtype == "f32":
        b = b.float()
        monkeypatch.setenv("CSRK_FUSED_DOT_F32", "1")  # fp32 runs unfused by default
    x_f, info_f = cg.cg(m, b, iters=40)
    x_f2, _ = cg.cg(m, b, iters=40)
    assert torch.equal(x_f, x_f2)
    monkeypatch.setenv("CSRK_NO_FUSED_DOT", "1")
    x_s, info_s = cg.cg(m, b, iters=40)
    tol = 1e-9 if dtype == "f64" else 1e-3
    assert (x_f.double() - x_s.double()).abs().max().item() <= tol * x_s.double().abs().max().item()
    if dtype == "f64":
        assert info_f["rr"] == pytest.approx(info_s["rr"], rel=1e-6)
