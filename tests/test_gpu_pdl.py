"""Back-to-back SpMVs under programmatic dependent launch (csrc/spmv.cu
launch_stream): the next launch's producer streams the matrix while the
previous grid finishes, and its consumers read x only after
griddepcontrol.wait.  The sharpest case is a chain y_{k+1} = A y_k with no
other kernel in between -- each launch reads exactly what the previous one
is still writing when it starts -- checked bit for bit against the oracle's
chain; plus resident replicas of one matrix (the bench's rotation for small
configs) giving identical y."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from oracle import oracle as O
from paper_2203_05096_b200 import _native as nat
from paper_2203_05096_b200 import synthetic

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _matrix(shape=(48, 48, 48), points=7):
    n, rp, ci, va = synthetic.stencil_arrays(shape, points)
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    return a, ck.pack_csrk(a, res.perm, res.level_group_sizes)


@pytest.mark.parametrize("variant,nx", [("serial", 1), ("strided", 4)])
def test_chained_spmv_back_to_back(variant, nx):
    a, m = _matrix()
    n = a.n_rows
    b = m.base
    x0 = np.random.default_rng(7).uniform(-1.0, 1.0, n)
    dims = ck.BlockDims(nx, 1, 1)
    steps = 8
    vs = [torch.from_numpy(x0).cuda()] + [torch.empty(n, dtype=torch.float64, device="cuda")
                                          for _ in range(steps)]
    stream = torch.cuda.current_stream()
    for k in range(steps):  # no kernel between two launches
        ck.spmv_device(m, vs[k], vs[k + 1], dims=dims, variant=variant, stream=stream)
    torch.cuda.synchronize()
    v = x0
    for k in range(steps):
        if variant == "serial":
            v = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, v)
        else:
            v = O.spmv_strided(b.row_ptr, b.col_idx, b.vals, v, nx)
        np.testing.assert_array_equal(vs[k + 1].cpu().numpy(), v)


def test_chained_spmv_in_place_pairs_f32():
    """ping-pong between two buffers in fp32: launch k + 1 overwrites the x
    of launch k, which must have finished reading it"""
    a, m = _matrix((40, 40, 40), 27)
    n = a.n_rows
    x0 = np.random.default_rng(8).uniform(-1.0, 1.0, n).astype(np.float32)
    p = torch.from_numpy(x0).cuda()
    q = torch.empty_like(p)
    for _ in range(6):
        ck.spmv_device(m, p, q)
        ck.spmv_device(m, q, p)
    torch.cuda.synchronize()
    got = p.cpu().numpy()
    # the same chain one launch at a time with a host round trip in between
    r = torch.from_numpy(x0).cuda()
    s = torch.empty_like(r)
    for _ in range(6):
        ck.spmv_device(m, r, s)
        torch.cuda.synchronize()
        ck.spmv_device(m, s, r)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(got, r.cpu().numpy())


def test_replicas_give_identical_y():
    a, m = _matrix((32, 32, 32))
    n = a.n_rows
    b = m.base
    x = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, n)).cuda()
    ys = []
    devs = [m.device()] + [nat.DeviceMatrix.upload(b.row_ptr, b.col_idx, b.vals, n, n, k=3,
                                                   sr_ptr=m.group_ptrs[0],
                                                   ssr_ptr=m.group_ptrs[1])
                           for _ in range(3)]
    for d in devs:
        ys.append(ck.spmv_device(d, x.clone()))
    torch.cuda.synchronize()
    want = O.spmv_grouped(O.csr3_group_rows(m.sr_ptr, m.ssr_ptr), b.row_ptr, b.col_idx,
                          b.vals, x.cpu().numpy(), 4)
    for y in ys:
        np.testing.assert_array_equal(y.cpu().numpy(), want)
