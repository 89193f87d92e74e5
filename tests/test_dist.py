"""Multi-GPU host logic on CPU: nnz-balanced SSR partition,
rank blocks, and both x exchanges over gloo with world_size 2 and 3; plus a
one-GPU loopback check that partitioned device SpMVs reassemble the global y
bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2203_05096_b200 as ck
from oracle import oracle as O
from paper_2203_05096_b200 import dist as D
from paper_2203_05096_b200 import synthetic


def _packed(shape=(20, 20, 20), points=7, targets=(8, 8)):
    n, rp, ci, va = synthetic.stencil_arrays(shape, points, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, list(targets))
    # the CPU tests build the packed arrays with the oracle (no GPU here)
    prp, pci, pva = O.permute_symmetric(rp, ci, va, res.perm.fwd, res.perm.inv)
    base = ck.CsrMatrix(n, n, prp, pci, pva)
    ptrs = (O.group_pointers(res.level_group_sizes[0]),
            O.group_pointers(res.level_group_sizes[1]))
    return ck.CsrKMatrix(base, 3, ptrs, res.perm)


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_is_ssr_aligned_and_balanced(parts):
    m = _packed()
    b = m.base
    cuts = D.partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, parts)
    assert cuts[0] == 0 and cuts[-1] == b.n_rows and np.all(np.diff(cuts) >= 0)
    ssr_rows = m.sr_ptr.astype(np.int64)[m.ssr_ptr.astype(np.int64)]
    assert set(cuts.tolist()) <= set(ssr_rows.tolist())
    rp = b.row_ptr.astype(np.int64)
    per = [int(rp[cuts[g + 1]] - rp[cuts[g]]) for g in range(parts)]
    max_ssr = int(np.diff(rp[ssr_rows]).max())
    assert max(per) - min(per) <= 2 * max_ssr
    # rank blocks reassemble the global product
    x = np.random.default_rng(0).uniform(-1, 1, b.n_rows)
    want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)
    got = []
    for g in range(parts):
        blk = D.local_block(m, int(cuts[g]), int(cuts[g + 1]))
        got.append(O.spmv_serial(blk.row_ptr, blk.col_idx, blk.vals, x))
    np.testing.assert_array_equal(np.concatenate(got), want)


def test_halo_plan_covers_footprints():
    m = _packed()
    b = m.base
    cuts = D.partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, 4)
    fps = D.footprints(b.row_ptr, b.col_idx, cuts)
    plan = D.halo_plan(cuts, fps)
    for dst in range(4):
        covered = np.zeros(b.n_rows, dtype=bool)
        covered[cuts[dst]:cuts[dst + 1]] = True
        for s, d, lo, hi in plan:
            if d == dst:
                assert cuts[s] <= lo < hi <= cuts[s + 1]
                covered[lo:hi] = True
        lo, hi = fps[dst]
        assert covered[lo:hi].all()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _packed()
        b = m.base
        cuts = D.partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, world)
        fps = D.footprints(b.row_ptr, b.col_idx, cuts)
        ex = D.Exchange(rank, world, cuts, fps, mode)
        x = np.random.default_rng(1).uniform(-1, 1, b.n_rows)
        x_full = torch.full((b.n_rows,), float("nan"), dtype=torch.float64)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        x_full[r0:r1] = torch.from_numpy(x[r0:r1])
        ex(x_full)
        lo, hi = fps[rank]
        ok_window = bool(torch.equal(x_full[lo:hi], torch.from_numpy(x[lo:hi])))
        blk = D.local_block(m, r0, r1)
        y_local = O.spmv_serial(blk.row_ptr, blk.col_idx, blk.vals,
                                np.nan_to_num(x_full.numpy(), nan=1e300))
        want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)[r0:r1]
        ok_y = bool(np.array_equal(y_local, want))
        result_q.put((rank, ok_window, ok_y, ex.bytes_received()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "halo"), (2, "allgather"), (3, "halo")])
def test_exchange_over_gloo(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_window, ok_y, nbytes in results:
        assert ok_window, f"rank {rank}: x footprint not filled by {mode}"
        assert ok_y, f"rank {rank}: local SpMV differs after {mode}"
        assert nbytes > 0


def _local_worker(rank, world, port, mode, result_q):
    """DistSpMV's host-side pieces on CPU tensors over gloo: the rank's block
    with footprint-local columns, the interior rows computed BEFORE the
    exchange (halo poisoned with NaN), the exchange, then the boundary rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _packed()
        b = m.base
        cuts = D.partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, world)
        fps = D.footprints(b.row_ptr, b.col_idx, cuts)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        lo, hi = (int(v) for v in fps[rank])
        x0, x1 = min(lo, r0), max(hi, r1)
        blk = D.local_block(m, r0, r1, col0=x0)
        x = np.random.default_rng(1).uniform(-1, 1, b.n_rows)
        x_local = torch.full((x1 - x0,), float("nan"), dtype=torch.float64)
        x_local[r0 - x0:r1 - x0] = torch.from_numpy(x[r0:r1])
        a, bb = D.interior_rows(blk.row_ptr, blk.col_idx, r0 - x0, r1 - x0)
        want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)[r0:r1]
        early = O.spmv_serial(blk.row_ptr, blk.col_idx, blk.vals, x_local.numpy())
        ok_interior = bool(np.array_equal(early[a:bb], want[a:bb]))
        ex = D.XExchange(rank, world, cuts, fps, x0, mode)
        ex.finish(x_local, ex.start(x_local))
        ok_window = bool(torch.equal(x_local, torch.from_numpy(x[x0:x1])))
        y = O.spmv_serial(blk.row_ptr, blk.col_idx, blk.vals, x_local.numpy())
        result_q.put((rank, ok_interior, ok_window, bool(np.array_equal(y, want)),
                      bb - a, r1 - r0, x1 - x0, ex.bytes_received()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "halo"), (2, "allgather"), (3, "halo"),
                                        (4, "halo"), (3, "allgather")])
def test_footprint_local_exchange_over_gloo(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_local_worker, args=(r, world, port, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = _packed().base.n_rows
    for rank, ok_int, ok_win, ok_y, n_int, n_own, n_loc, nbytes in results:
        assert ok_int, f"rank {rank}: interior rows read the halo"
        assert ok_win, f"rank {rank}: footprint x not filled by {mode}"
        assert ok_y, f"rank {rank}: local SpMV differs"
        assert n_loc < n, "local x must be footprint-sized, not global"
        assert 0 <= n_int <= n_own
    assert sum(r[4] for r in results) > 0  # (a narrow middle block may be all halo)


def test_interior_rows_edge_cases():
    # rows: [own only], [reads below], [empty], [reads above]
    rp = np.array([0, 2, 4, 4, 6], dtype=np.uint32)
    ci = np.array([5, 6, 3, 7, 6, 12], dtype=np.uint32)
    assert D.interior_rows(rp, ci, 5, 10) == (2, 3)
    assert D.interior_rows(rp, ci, 0, 20) == (0, 4)
    assert D.interior_rows(np.zeros(1, np.uint32), np.zeros(0, np.uint32), 0, 1) == (0, 0)


@pytest.mark.gpu
def test_partitioned_device_spmv_reassembles_bitwise():
    from paper_2203_05096_b200 import _native as nat
    n, rp, ci, va = synthetic.stencil_arrays((32, 32, 32), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    x = np.random.default_rng(3).uniform(-1, 1, n)
    want = ck.spmv_csr3(m, x)
    for parts in (2, 3, 8):
        cuts = D.partition_by_nnz(m.base.row_ptr, m.sr_ptr, m.ssr_ptr, parts)
        ys = []
        for g in range(parts):
            blk = D.local_block(m, int(cuts[g]), int(cuts[g + 1]))
            dev = nat.DeviceMatrix.upload(blk.row_ptr, blk.col_idx, blk.vals,
                                          blk.r1 - blk.r0, n, k=3, sr_ptr=blk.sr_ptr,
                                          ssr_ptr=blk.ssr_ptr)
            ys.append(dev.spmv_host(x) if blk.r1 > blk.r0 else np.zeros(0))
        np.testing.assert_array_equal(np.concatenate(ys), want)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,nx", [("serial", 1), ("strided", 4)])
def test_dist_blocks_interior_then_boundary_bitwise(variant, nx):
    """DistSpMV's device part on one GPU, rank by rank: footprint-local x
    with a NaN halo, the interior tiles (they must not read the halo), then
    the halo filled (what the exchange delivers) and the boundary tiles --
    the slices reassemble the single-GPU y bit for bit."""
    n, rp, ci, va = synthetic.stencil_arrays((40, 40, 40), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    b = m.base
    x = np.random.default_rng(5).uniform(-1, 1, n)
    want = (O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x) if variant == "serial"
            else O.spmv_strided(b.row_ptr, b.col_idx, b.vals, x, nx))
    for parts in (1, 2, 3, 8):
        got = []
        interior_seen = 0
        for g in range(parts):
            op = D.DistSpMV(m, g, parts, variant=variant, nx=nx)
            xl = torch.full((op.n_local_cols,), float("nan"), dtype=torch.float64,
                            device="cuda")
            xl[op.own] = torch.from_numpy(x[op.r0:op.r1]).cuda()
            y = torch.full((op.n_own,), float("nan"), dtype=torch.float64, device="cuda")
            s = torch.cuda.current_stream().cuda_stream
            op._tiles(xl, y, op.t_lo, op.t_hi, s)
            torch.cuda.synchronize()
            tr = op.dev.tile_rows()
            ra, rb = int(tr[op.t_lo]), int(tr[op.t_hi])
            np.testing.assert_array_equal(y[ra:rb].cpu().numpy(), want[op.r0 + ra:op.r0 + rb])
            interior_seen += rb - ra
            xl.copy_(torch.from_numpy(x[op.x0:op.x1]).cuda())
            op._tiles(xl, y, 0, op.t_lo, s)
            op._tiles(xl, y, op.t_hi, op.n_tiles, s)
            torch.cuda.synchronize()
            got.append(y.cpu().numpy())
            assert op.n_local_cols < n or parts == 1
        np.testing.assert_array_equal(np.concatenate(got), want)
        assert interior_seen > 0


def _host_slab(shape, points, lay, values="uniform"):
    """The rows of a slab from the host generator, columns shifted to the
    slab's local x (what csrk_stencil_slab writes with Laplacian values)."""
    n, rp, ci, va = synthetic.stencil_arrays(shape, points, values=values)
    r0, r1 = lay.global_row0, lay.global_row0 + lay.n_own
    p0, p1 = int(rp[r0]), int(rp[r1])
    base = lay.global_row0 - lay.own_off
    return ((rp[r0:r1 + 1] - p0).astype(np.uint32), (ci[p0:p1] - base).astype(np.uint32),
            va[p0:p1], (n, rp, ci, va))


@pytest.mark.parametrize("nz,world", [(1, 1), (7, 1), (7, 2), (8, 3), (9, 9), (16, 5)])
def test_slab_layout(nz, world):
    shape = (nz, 3, 4)
    lays = [D.SlabLayout.of(shape, g, world) for g in range(world)]
    assert sum(l.n_own for l in lays) == nz * 12
    assert lays[0].global_row0 == 0 and not lays[0].has_lo and not lays[-1].has_hi
    for g, lay in enumerate(lays):
        assert lay.n_own >= 12
        assert lay.n_cols == lay.n_own + 12 * (int(g > 0) + int(g < world - 1))
        a, b = lay.interior_rows()
        assert 0 <= a <= b <= lay.n_own
        rp, ci, _, _ = _host_slab(shape, 7, lay)
        assert int(ci.max()) < lay.n_cols
        for r in range(lay.n_own):  # interior rows read owned x only
            cols = ci[rp[r]:rp[r + 1]]
            inside = (cols >= lay.own_off).all() and (cols < lay.own_off + lay.n_own).all()
            if a <= r < b:
                assert inside
    with pytest.raises(ValueError):
        D.slab_cuts(2, 3)


def test_interior_tiles():
    tr = np.array([0, 5, 9, 14, 20, 26, 30])
    assert D.interior_tiles(tr, 5, 26) == (1, 5)
    assert D.interior_tiles(tr, 6, 25) == (2, 4)
    assert D.interior_tiles(tr, 0, 30) == (0, 6)
    assert D.interior_tiles(tr, 10, 12) == (3, 3)


def _slab_worker(rank, world, port, shape, points, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = D.SlabLayout.of(shape, rank, world)
        rp, ci, va, (n, grp, gci, gva) = _host_slab(shape, points, lay)
        x = np.random.default_rng(7).uniform(-1, 1, n)
        x_local = torch.full((lay.n_cols,), float("nan"), dtype=torch.float64)
        g0 = lay.global_row0
        x_local[lay.own_off:lay.own_off + lay.n_own] = torch.from_numpy(x[g0:g0 + lay.n_own])
        ex = D.SlabExchange(lay)
        ex(x_local)
        base = g0 - lay.own_off
        ok_x = bool(torch.equal(x_local, torch.from_numpy(x[base:base + lay.n_cols])))
        y = O.spmv_serial(rp, ci, va, x_local.numpy())
        want = O.spmv_serial(grp, gci, gva, x)[g0:g0 + lay.n_own]
        result_q.put((rank, ok_x, bool(np.array_equal(y, want)), ex.bytes_received()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,points", [(2, (6, 5, 4), 7), (3, (7, 4, 5), 27)])
def test_slab_exchange_over_gloo(world, shape, points):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, shape, points, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_x, ok_y, nbytes in results:
        assert ok_x, f"rank {rank}: halo planes not filled"
        assert ok_y, f"rank {rank}: slab SpMV differs from the global rows"
        assert nbytes == 8 * shape[1] * shape[2] * (int(rank > 0) + int(rank < world - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("points", [7, 27])
def test_device_slabs_reassemble_bitwise(points):
    """csrk_stencil_slab equals the host rows bit for bit, and the per-rank
    interior + boundary tile launches reassemble the global y."""
    shape = (23, 17, 19)
    n, rp, ci, va = synthetic.stencil_arrays(shape, points, values="laplacian")
    x = np.random.default_rng(11).uniform(-1, 1, n)
    want = O.spmv_serial(rp, ci, va, x)
    for world in (1, 2, 3, 5):
        ys = []
        for g in range(world):
            op = D.SlabSpMV(shape, points, g, world)
            lay = op.lay
            hrp, hci, hva, _ = _host_slab(shape, points, lay, values="laplacian")
            drp, dci, dva, _, _ = op.dev.download()
            np.testing.assert_array_equal(drp, hrp)
            np.testing.assert_array_equal(dci, hci)
            np.testing.assert_array_equal(dva, hva)
            base = lay.global_row0 - lay.own_off
            xl = torch.from_numpy(x[base:base + lay.n_cols].copy()).cuda()
            y = torch.empty(lay.n_own, dtype=torch.float64, device="cuda")
            op.compute(xl, y)
            torch.cuda.synchronize()
            ys.append(y.cpu().numpy())
        np.testing.assert_array_equal(np.concatenate(ys), want)


class _HostSlabOp:
    """CPU stand-in for SlabSpMV (exchange over gloo, oracle SpMV)."""

    def __init__(self, shape, points, rank, world):
        self.lay = D.SlabLayout.of(shape, rank, world)
        self.rp, self.ci, self.va, _ = _host_slab(shape, points, self.lay)
        self.ex = D.SlabExchange(self.lay)
        self.own = slice(self.lay.own_off, self.lay.own_off + self.lay.n_own)
        self.n_own = self.lay.n_own
        self.n_local_cols = self.lay.n_cols
        self.launches_per_step = 1

    def step(self, x_local, y_own):
        if self.lay.world > 1:
            self.ex(x_local)
        y_own.copy_(torch.from_numpy(O.spmv_serial(self.rp, self.ci, self.va,
                                                   x_local.numpy())))
        return y_own


class _HostCgSteps:
    """CPU stand-in for dist.DeviceCgSteps: the same step semantics (the
    reduction folded into sc, rr published by the direction step)."""

    def __init__(self):
        self.sc = torch.zeros(8, dtype=torch.float64)

    def dot(self, a, b, slot):
        self.sc[slot] = torch.dot(a.double(), b.double())

    def update(self, x, r, p, ap):
        pap = float(self.sc[1])
        alpha = float(self.sc[0]) / pap if pap != 0.0 else 0.0
        x.add_(p, alpha=alpha)
        r.add_(ap, alpha=-alpha)
        self.sc[2] = torch.dot(r.double(), r.double())

    def direction(self, p, r):
        rr, rr_new = float(self.sc[0]), float(self.sc[2])
        beta = rr_new / rr if rr != 0.0 else 0.0
        p.mul_(beta).add_(r)
        self.sc[0] = rr_new


def _cg_worker(rank, world, port, shape, iters, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = _HostSlabOp(shape, 7, rank, world)
        n = shape[0] * shape[1] * shape[2]
        b = np.random.default_rng(5).uniform(-1, 1, n)
        g0 = op.lay.global_row0
        b_own = torch.from_numpy(b[g0:g0 + op.lay.n_own].copy())
        x_own = torch.zeros_like(b_own)
        x_own, rr = D.DistCG(op, steps=_HostCgSteps()).run(b_own, x_own, iters)
        result_q.put((rank, g0, x_own.numpy(), float(rr.item())))
    finally:
        dist.destroy_process_group()


def _numpy_cg(shape, b, iters):
    n, rp, ci, va = synthetic.stencil_arrays(shape, 7, values="uniform")
    a = lambda v: O.spmv_serial(rp, ci, va, v)  # noqa: E731
    x = np.zeros(n)
    r = b - a(x)
    p = r.copy()
    rr = r @ r
    for _ in range(iters):
        ap = a(p)
        alpha = rr / (p @ ap)
        x += alpha * p
        r -= alpha * ap
        rr_new = r @ r
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, rr


@pytest.mark.parametrize("world", [1, 2, 3])
def test_dist_cg_over_gloo(world):
    """Slab-partitioned CG (halo planes + all-reduced dots) equals one-process
    CG on the whole matrix to rounding."""
    shape, iters = (9, 6, 5), 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cg_worker, args=(r, world, port, shape, iters, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.concatenate([t[2] for t in results])
    b = np.random.default_rng(5).uniform(-1, 1, x.size)
    want, rr = _numpy_cg(shape, b, iters)
    np.testing.assert_allclose(x, want, rtol=1e-9, atol=1e-12)
    assert all(abs(t[3] - rr) <= 1e-9 * max(rr, 1e-300) + 1e-300 for t in results)


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["C2", "C2-torch", "C2-slab", "C4"])
def test_bench_multi_gpu_path_one_rank(config):
    """bench.py's torchrun path (NCCL process group, SSR row blocks with the
    halo exchange and the oracle parity check, the slab partition, the
    distributed CG) end to end with one rank (CSRK_DIST=1): the JSON line
    has the contract's keys and the weak / strong labels."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "1",
           "--steps", "3", "--warmup", "3", "--config", config.split("-")[0]]
    if config == "C2-slab":
        cmd += ["--partition", "slab"]
    if config == "C2-torch":
        cmd += ["--mg", "torch"]
    if config == "C4":
        cmd += ["--side", "96", "--iters", "10"]
    env = dict(os.environ, CSRK_DIST="1")
    out = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "scaling", "e2e",
                "roofline", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert line["scaling"] == ("weak" if config == "C2-slab" else "strong")
    if config in ("C2", "C2-torch"):
        assert line["parity"]["ok"] and line["efficiency_t1_over_n_tn"] > 0
        # default: the C-ABI path with its timed steps in one CUDA graph
        assert line["timed_as"] == ("K eager steps" if config == "C2-torch"
                                    else "one CUDA graph of the K steps")
    assert line["e2e"]["h2d_bytes_per_step"] > 0
    if config == "C4":
        assert line["timed_as"] == "one CUDA graph per step"


@pytest.mark.gpu
@pytest.mark.parametrize("chunks,nz", [(1, 40), (3, 40), (8, 40), (8, 6), (5, 5)])
def test_slab_host_pipeline_bitwise(chunks, nz):
    """SlabSpMV.step_host (chunked H2D / interior tiles / D2H on three
    streams) gives the bits of the device-resident step (one rank),
    including one-plane chunks whose tiles read two chunks ahead."""
    shape = (nz, 48, 56)
    op = D.SlabSpMV(shape, 7, 0, 1)
    lay = op.lay
    x = torch.from_numpy(np.random.default_rng(chunks).uniform(-1, 1, lay.n_own))
    x_local = torch.zeros(lay.n_cols, dtype=torch.float64, device="cuda")
    y = torch.empty(lay.n_own, dtype=torch.float64, device="cuda")
    x_local[lay.own_off:lay.own_off + lay.n_own] = x.cuda()
    op.compute(x_local, y)
    torch.cuda.synchronize()
    want = y.cpu().numpy().copy()
    x_pin = x.clone().pin_memory()
    y_pin = torch.full((lay.n_own,), float("nan"), dtype=torch.float64).pin_memory()
    x_local.zero_()
    for _ in range(2):
        op.step_host(x_pin, y_pin, x_local, y, chunks=chunks)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y_pin.numpy(), want)


def test_bench_gpus_flag_relaunches_under_torchrun():
    """`python bench.py --gpus N` without torchrun re-launches itself as N
    ranks (torch.distributed.run); rank 0 prints the one JSON line."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "3", "--probe-launch"],
                         cwd=repo, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["world_size"] == 3 and line["n_gpus"] == 3 and line["torchrun"]


# ---- the multi-GPU C-ABI (csrk_mg_*) -----------------------

@pytest.mark.parametrize("parts", [1, 2, 3, 5, 8])
def test_native_mg_planning_matches_dist(parts):
    """csrk_mg_partition / csrk_mg_footprints / csrk_mg_plan (host C++, no
    GPU) equal dist.partition_by_nnz / footprints / halo_plan."""
    for shape, points, targets in (((20, 20, 20), 7, (8, 8)), ((12, 12, 12), 27, (4, 8))):
        m = _packed(shape, points, targets)
        b = m.base
        cuts = D.partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, parts)
        np.testing.assert_array_equal(D.native_partition(m, parts), cuts)
        fps = D.footprints(b.row_ptr, b.col_idx, cuts)
        np.testing.assert_array_equal(D.native_footprints(b.row_ptr, b.col_idx, cuts), fps)
        assert D.native_halo_plan(cuts, fps) == D.halo_plan(cuts, fps)


def test_native_mg_partition_rejects_bad_parts():
    m = _packed((8, 8, 8), 7, (4, 4))
    with pytest.raises(ValueError, match="parts"):
        D.native_partition(m, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,nx", [("serial", 1), ("strided", 4)])
def test_native_mg_blocks_bitwise(variant, nx):
    """csrk_mg_* on one GPU: world 1 with its own NCCL communicator (no
    transfers) equals the single-GPU y; world 2 / 3 / 8 rank by rank without
    a communicator (halo pre-filled, as the exchange delivers it) -- same
    interior tile split as DistSpMV, slices reassemble the y bit for bit."""
    n, rp, ci, va = synthetic.stencil_arrays((40, 40, 40), 7, values="uniform")
    a = ck.CsrMatrix(n, n, rp, ci, va)
    res = ck.band_k(a, 3, [8, 8])
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    b = m.base
    x = np.random.default_rng(7).uniform(-1, 1, n)
    want = (O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x) if variant == "serial"
            else O.spmv_strided(b.row_ptr, b.col_idx, b.vals, x, nx))
    op = D.NativeDistSpMV(m, 0, 1, variant=variant, nx=nx)
    xl = torch.from_numpy(x).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    op.step(xl, y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), want)
    assert op.info()["sent"] == 0 and op.info()["t_hi"] == op.info()["n_tiles"]
    op.close()
    for parts in (2, 3, 8):
        got = []
        for g in range(parts):
            nd = D.NativeDistSpMV(m, g, parts, variant=variant, nx=nx, communicator=False)
            py = D.DistSpMV(m, g, parts, variant=variant, nx=nx)
            xl = torch.from_numpy(x[nd.x0:nd.x1]).cuda()
            yo = torch.full((nd.n_own,), float("nan"), dtype=torch.float64, device="cuda")
            nd.step(xl, yo)
            torch.cuda.synchronize()
            info = nd.info()
            assert (info["t_lo"], info["t_hi"], info["n_tiles"]) == (py.t_lo, py.t_hi,
                                                                     py.n_tiles)
            assert info["received"] == sum(hi - lo for _, lo, hi in py.exchange.recvs)
            got.append(yo.cpu().numpy())
            nd.close()
        np.testing.assert_array_equal(np.concatenate(got), want)


@pytest.mark.gpu
def test_dist_cg_graph_replay_equals_eager_one_rank():
    """DistCG.graphed (SpMV launches, step kernels and, at N > 1, the halo
    and the all-reduces captured into one CUDA graph) gives the eager run's
    bits; one rank, no process group."""
    op = D.SlabSpMV((24, 24, 24), 7, 0, 1)
    n = op.lay.n_own
    b = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, n)).cuda()
    solver = D.DistCG(op)
    x_e = torch.zeros_like(b)
    solver.run(b, x_e, 20)
    x_g = torch.zeros_like(b)
    g = solver.graphed(b, x_g, 20)
    x_g.fill_(123.0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x_g, x_e)
