"""Multi-GPU CSR-k SpMV: row-block partition of super-super-rows, x exchange.

SURVEY.md §8(e).  One process per GPU (torchrun), ``torch.distributed`` over
NCCL for the plumbing.  The matrix is split at super-super-row boundaries so
every rank holds a contiguous row block with about the same number of
nonzeros (the reference's static chunks, kernels.py:150-155, generalised from
equal group counts to equal nonzeros).  Rows keep their global column
indices; every rank keeps a full-length x buffer whose owned slice it
updates itself, and before each SpMV the rest of its column footprint is
filled by one of two exchanges:

  "halo"       (default) ``batch_isend_irecv`` of exactly the contiguous x
               windows each rank's rows read from each peer; with Band-k
               ordering these are narrow bands next to the owned slice;
  "allgather"  the literal north-star collective: every rank's owned slice
               (padded to the largest) all-gathered, then copied into place.

y slices are disjoint, so no reduction is needed.  The exchange code only
uses tensor slicing and torch.distributed, so it runs unchanged on CPU
tensors over gloo (tests/test_dist.py) and on CUDA tensors over NCCL.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "partition_by_nnz",
    "footprints",
    "halo_plan",
    "RankBlock",
    "local_block",
    "Exchange",
    "DistSpMV",
    "bench_main",
]


def partition_by_nnz(row_ptr, sr_ptr, ssr_ptr, n_parts: int) -> np.ndarray:
    """Row cuts (n_parts + 1 entries) on super-super-row boundaries that
    balance nonzeros: part g starts at the first SSR whose starting nonzero
    offset reaches g * nnz / n_parts."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    ssr_rows = np.asarray(sr_ptr, dtype=np.int64)[np.asarray(ssr_ptr, dtype=np.int64)]
    nnz_at = rp[ssr_rows]  # nonzero offset at every SSR start (and the end)
    total = int(rp[-1])
    cuts = [0]
    for g in range(1, n_parts):
        target = (total * g + n_parts - 1) // n_parts
        s = int(np.searchsorted(nnz_at, target, side="left"))
        cuts.append(int(ssr_rows[min(s, len(ssr_rows) - 1)]))
    cuts.append(int(ssr_rows[-1]))
    cuts = np.maximum.accumulate(np.asarray(cuts, dtype=np.int64))
    return cuts


def footprints(row_ptr, col_idx, cuts) -> np.ndarray:
    """(lo, hi) column range read by each part's rows (hi exclusive;
    lo = hi = row start for an empty part)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx)
    out = np.zeros((len(cuts) - 1, 2), dtype=np.int64)
    for g in range(len(cuts) - 1):
        a, b = int(rp[cuts[g]]), int(rp[cuts[g + 1]])
        if b > a:
            seg = ci[a:b]
            out[g] = (int(seg.min()), int(seg.max()) + 1)
        else:
            out[g] = (cuts[g], cuts[g])
    return out


def halo_plan(cuts, fps) -> list:
    """Transfers (src, dst, lo, hi): dst needs x[lo:hi] owned by src."""
    plan = []
    g_count = len(cuts) - 1
    for dst in range(g_count):
        lo, hi = fps[dst]
        for src in range(g_count):
            if src == dst:
                continue
            a, b = max(lo, cuts[src]), min(hi, cuts[src + 1])
            if b > a:
                plan.append((src, dst, int(a), int(b)))
    return plan


@dataclass
class RankBlock:
    """The rows [r0, r1) of a packed CSR-k matrix as a standalone CSR-k with
    global column indices (local row / group numbering)."""

    r0: int
    r1: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    sr_ptr: np.ndarray
    ssr_ptr: np.ndarray


def local_block(m, r0: int, r1: int) -> RankBlock:
    """Slice a CsrKMatrix (k = 3) at SSR-aligned rows [r0, r1)."""
    b = m.base
    rp = b.row_ptr.astype(np.int64)
    p0, p1 = int(rp[r0]), int(rp[r1])
    sr = m.sr_ptr.astype(np.int64)
    ssr = m.ssr_ptr.astype(np.int64)
    s0, s1 = int(np.searchsorted(sr, r0)), int(np.searchsorted(sr, r1))
    q0, q1 = int(np.searchsorted(ssr, s0)), int(np.searchsorted(ssr, s1))
    if sr[s0] != r0 or sr[s1] != r1 or ssr[q0] != s0 or ssr[q1] != s1:
        raise ValueError("rank block must start and end on super-super-row boundaries")
    return RankBlock(
        r0=r0, r1=r1, n_cols=b.n_cols,
        row_ptr=(rp[r0:r1 + 1] - p0).astype(np.uint32),
        col_idx=b.col_idx[p0:p1], vals=b.vals[p0:p1],
        sr_ptr=(sr[s0:s1 + 1] - r0).astype(np.uint32),
        ssr_ptr=(ssr[q0:q1 + 1] - s0).astype(np.uint32))


class Exchange:
    """x exchange of one rank on a full-length x buffer (any device)."""

    def __init__(self, rank: int, world: int, cuts, fps, mode: str = "halo", group=None):
        if mode not in ("halo", "allgather"):
            raise ValueError(f"unknown exchange mode {mode!r}")
        self.rank, self.world, self.mode, self.group = rank, world, mode, group
        self.cuts = [int(c) for c in cuts]
        plan = halo_plan(self.cuts, fps)
        self.sends = [(d, a, b) for s, d, a, b in plan if s == rank]
        self.recvs = [(s, a, b) for s, d, a, b in plan if d == rank]
        self.maxlen = max(self.cuts[g + 1] - self.cuts[g] for g in range(world))
        self._gather = None

    def bytes_received(self, itemsize: int = 8) -> int:
        if self.mode == "allgather":
            return (self.world - 1) * self.maxlen * itemsize
        return sum(b - a for _, a, b in self.recvs) * itemsize

    def __call__(self, x_full):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return x_full
        if self.mode == "halo":
            ops = [dist.P2POp(dist.isend, x_full[a:b], d, group=self.group)
                   for d, a, b in self.sends]
            ops += [dist.P2POp(dist.irecv, x_full[a:b], s, group=self.group)
                    for s, a, b in self.recvs]
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            return x_full
        lo, hi = self.cuts[self.rank], self.cuts[self.rank + 1]
        if self._gather is None or self._gather[0].device != x_full.device:
            self._gather = [torch.zeros(self.maxlen, dtype=x_full.dtype, device=x_full.device)
                            for _ in range(self.world)]
        mine = self._gather[self.rank]
        mine[: hi - lo].copy_(x_full[lo:hi])
        dist.all_gather(self._gather, mine.clone(), group=self.group)
        for g in range(self.world):
            a, b = self.cuts[g], self.cuts[g + 1]
            if g != self.rank and b > a:
                x_full[a:b].copy_(self._gather[g][: b - a])
        return x_full


class DistSpMV:
    """y_local = A[r0:r1, :] x on this rank's GPU after the x exchange."""

    def __init__(self, m, rank: int, world: int, mode: str = "halo", group=None,
                 device=None, f32: bool = False):
        from . import _native as nat

        b = m.base
        self.cuts = partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, world)
        self.fps = footprints(b.row_ptr, b.col_idx, self.cuts)
        self.rank, self.world = rank, world
        self.r0, self.r1 = int(self.cuts[rank]), int(self.cuts[rank + 1])
        blk = local_block(m, self.r0, self.r1)
        self.nnz_local = int(blk.row_ptr[-1])
        self.nnz_total = b.nnz
        self.n = b.n_rows
        self.dev = nat.DeviceMatrix.upload(
            blk.row_ptr, blk.col_idx, blk.vals, self.r1 - self.r0, b.n_cols, k=3,
            sr_ptr=blk.sr_ptr, ssr_ptr=blk.ssr_ptr, device=device, f32=f32)
        self.exchange = Exchange(rank, world, self.cuts, self.fps, mode, group)
        self.f32 = f32

    def step(self, x_full, y_local, stream=None, dims=None, strided=False):
        """Exchange x then run the local SpMV (stream-ordered)."""
        import torch

        from . import _native as nat

        self.exchange(x_full)
        if self.r1 > self.r0:
            s = stream or torch.cuda.current_stream(x_full.device)
            self.dev.spmv_ptr(x_full.data_ptr(), y_local.data_ptr(), s.cuda_stream,
                              variant=nat.CSRK_STRIDED if strided else nat.CSRK_SERIAL,
                              nx=dims.x if (strided and dims) else 1, f32=self.f32)
        return y_local


def _cached_build(cfg: str, rank: int, log):
    """Rank 0 builds the packed matrix and writes it to a cache file; the
    other ranks load it (one Band-k per job instead of one per rank)."""
    import torch.distributed as dist

    import paper_2203_05096_b200 as ck

    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"csrk_bench_{cfg}_{os.getpid()}")
    obj = [path]
    dist.broadcast_object_list(obj, src=0)
    path = obj[0] + ".npz"
    if rank == 0:
        import bench as _bench  # the driver script's builder

        a, m, xp, params, bt = _bench.build_matrix(cfg, log)
        np.savez(path, row_ptr=m.base.row_ptr, col_idx=m.base.col_idx, vals=m.base.vals,
                 sr_ptr=m.sr_ptr, ssr_ptr=m.ssr_ptr, fwd=m.perm.fwd, xp=xp,
                 params=np.array([params.ssrs, params.srs]))
    dist.barrier()
    z = np.load(path)
    n = len(z["row_ptr"]) - 1
    base = ck.CsrMatrix(n, n, z["row_ptr"], z["col_idx"], z["vals"], _trusted=True)
    perm = ck.Permutation.from_forward(z["fwd"])
    m = ck.CsrKMatrix(base, 3, (z["sr_ptr"], z["ssr_ptr"]), perm, _trusted=True)
    xp = z["xp"]
    dist.barrier()
    if rank == 0:
        os.remove(path)
    return m, xp, [int(v) for v in z["params"]]


def bench_main(args, log):
    """bench.py --gpus N under torchrun: halo exchange + local SpMV per step,
    device time max-reduced over ranks."""
    import torch
    import torch.distributed as dist

    from .bench import spmv_bytes

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    from . import _native as nat
    nat.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m, xp, (ssrs, srs) = _cached_build(args.config, rank, log)
    mode = os.environ.get("CSRK_EXCHANGE", "halo")
    op = DistSpMV(m, rank, world, mode=mode, device=local, f32=args.fp32)
    dtype = torch.float32 if args.fp32 else torch.float64
    x_full = torch.zeros(op.n, dtype=dtype, device="cuda")
    x_full[op.r0:op.r1] = torch.from_numpy(xp[op.r0:op.r1]).to("cuda", dtype)
    y = torch.empty(max(1, op.r1 - op.r0), dtype=dtype, device="cuda")
    for _ in range(args.warmup):
        op.step(x_full, y)
    torch.cuda.synchronize()
    dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        op.step(x_full, y)
    ev1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    ms = float(ms.item())
    vbytes = 4 if args.fp32 else 8
    gflops = 2.0 * op.nnz_total / (ms * 1e-3) / 1e9
    line = None
    if rank == 0:
        algo = spmv_bytes(op.n, op.n, op.nnz_total, vbytes)
        line = {
            "metric": "SpMV GFLOP/s and achieved HBM GB/s (% of peak) at 1/2/4/8 B200 vs host CPU",
            "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.fp32 else "f64",
            "data": "synthetic (deterministic grid Laplacian, x ~ U[-1,1) seed 0)",
            "config": {"workload": args.config, "n_rows": op.n, "nnz": op.nnz_total,
                       "parallelism": f"row-block SSR partition x{world}, {mode} x exchange",
                       "exchange_bytes_rank0": op.exchange.bytes_received(vbytes),
                       "ssrs_target": ssrs, "srs_target": srs},
            "aggregate_hbm_gbs": round(algo / (ms * 1e-3) / 1e9, 1),
            "gpu_launches": args.steps,
        }
    dist.destroy_process_group()
    return line
