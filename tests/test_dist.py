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
