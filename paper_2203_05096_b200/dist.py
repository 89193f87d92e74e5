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

Generated 3D stencils partition as z-slabs instead (``SlabSpMV``): each rank
generates its own planes in HBM (csrk_stencil_slab) with columns local to
[lower halo plane | own planes | upper halo plane], so no rank holds the
global matrix or a global-length x.  One step sends the first / last owned
plane to the neighbours (NCCL send / recv over NVLink) while the interior
tiles -- rows whose stencil stays inside the owned planes -- are computed,
then computes the two boundary planes.  This is the partition of the
weak-scaling bench (a C2-sized slab per GPU) and of the multi-GPU CG (C4).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "slab_cuts",
    "SlabLayout",
    "interior_tiles",
    "SlabExchange",
    "SlabSpMV",
    "DistCG",
    "DeviceCgSteps",
    "partition_by_nnz",
    "footprints",
    "halo_plan",
    "RankBlock",
    "local_block",
    "interior_rows",
    "XExchange",
    "Exchange",
    "DistSpMV",
    "bench_main",
]


def slab_cuts(nz: int, world: int) -> list:
    """Plane cuts: rank g owns planes [cuts[g], cuts[g + 1]).  Equal plane
    counts (+-1) balance nonzeros to within one plane."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} planes over {world} ranks")
    return [nz * g // world for g in range(world + 1)]


@dataclass(frozen=True)
class SlabLayout:
    """Local index spaces of one rank's slab of an nz x ny x nx grid."""

    nz: int
    ny: int
    nx: int
    rank: int
    world: int
    z0: int
    z1: int

    @classmethod
    def of(cls, shape, rank: int, world: int) -> "SlabLayout":
        nz, ny, nx = (int(v) for v in shape)
        cuts = slab_cuts(nz, world)
        return cls(nz, ny, nx, rank, world, cuts[rank], cuts[rank + 1])

    @property
    def plane(self) -> int:
        return self.ny * self.nx

    @property
    def has_lo(self) -> bool:
        return self.z0 > 0

    @property
    def has_hi(self) -> bool:
        return self.z1 < self.nz

    @property
    def n_own(self) -> int:
        """rows of this rank (and entries of its y)"""
        return (self.z1 - self.z0) * self.plane

    @property
    def own_off(self) -> int:
        """offset of the owned x entries in the local x"""
        return self.plane if self.has_lo else 0

    @property
    def n_cols(self) -> int:
        """length of the local x: own planes plus the halo planes"""
        return self.n_own + self.plane * (int(self.has_lo) + int(self.has_hi))

    @property
    def global_row0(self) -> int:
        return self.z0 * self.plane

    def interior_rows(self) -> tuple:
        """[a, b): local rows whose 7- / 27-point stencil reads owned x only"""
        a = self.plane if self.has_lo else 0
        b = self.n_own - (self.plane if self.has_hi else 0)
        return a, max(a, b)


def interior_tiles(tile_rows, a: int, b: int) -> tuple:
    """[t_lo, t_hi): the tiles whose rows all lie in [a, b)."""
    tr = np.asarray(tile_rows, dtype=np.int64)
    t_lo = int(np.searchsorted(tr, a, side="left"))
    t_hi = int(np.searchsorted(tr, b, side="right")) - 1
    return t_lo, max(t_lo, t_hi)


class SlabExchange:
    """Halo planes of a slab's local x: the first owned plane goes to
    rank - 1 (its upper halo), the last to rank + 1 (its lower halo)."""

    def __init__(self, layout: SlabLayout, group=None):
        self.lay, self.group = layout, group

    def bytes_received(self, itemsize: int = 8) -> int:
        return self.lay.plane * itemsize * (int(self.lay.has_lo) + int(self.lay.has_hi))

    def start(self, x_local) -> list:
        """Post the sends / receives (asynchronous); returns the works."""
        import torch.distributed as dist

        lay, p = self.lay, self.lay.plane
        ops = []
        if lay.has_lo:
            ops.append(dist.P2POp(dist.isend, x_local[lay.own_off:lay.own_off + p],
                                  lay.rank - 1, group=self.group))
            ops.append(dist.P2POp(dist.irecv, x_local[0:p], lay.rank - 1, group=self.group))
        if lay.has_hi:
            hi = lay.own_off + lay.n_own
            ops.append(dist.P2POp(dist.isend, x_local[hi - p:hi], lay.rank + 1,
                                  group=self.group))
            ops.append(dist.P2POp(dist.irecv, x_local[hi:hi + p], lay.rank + 1,
                                  group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def __call__(self, x_local):
        for w in self.start(x_local):
            w.wait()
        return x_local


class SlabSpMV:
    """y_own = A[own rows, :] x on this rank's slab of a generated 3D stencil
    (natural order, uniform srs / ssrs groups, k = 3)."""

    def __init__(self, shape, points: int, rank: int, world: int, srs: int = 8,
                 ssrs: int = 8, device=None, f32: bool = False, group=None):
        from . import synthetic

        self.lay = SlabLayout.of(shape, rank, world)
        lay = self.lay
        self.dev = synthetic.device_slab((lay.nz, lay.ny, lay.nx), points, lay.z0, lay.z1,
                                         device=device).group_uniform(srs, ssrs)
        if self.dev.n_cols != lay.n_cols or self.dev.n_rows != lay.n_own:
            raise AssertionError("slab generator and layout disagree")
        if f32:
            self.dev.ensure_f32()
        self.f32 = f32
        self.nnz_local = self.dev.nnz
        self.n_tiles = self.dev.plan()["n_tiles"]
        self.t_lo, self.t_hi = interior_tiles(self.dev.tile_rows(), *lay.interior_rows())
        self.exchange = SlabExchange(lay, group)
        self._pipe = None
        self.own = slice(lay.own_off, lay.own_off + lay.n_own)
        self.n_own = lay.n_own
        self.n_local_cols = lay.n_cols

    def step(self, x_local, y_own):
        """Exchange the halo planes while the interior tiles run, then the
        boundary tiles, ordered on the current stream (the NCCL works wait on
        it and it waits on them)."""
        import torch

        works = self.exchange.start(x_local) if self.lay.world > 1 else []
        return self.compute(x_local, y_own, works)

    def compute(self, x_local, y_own, works=()):
        """Interior tiles, then wait for ``works`` (the halo), then the
        boundary tiles; a complete local x needs no works."""
        import torch

        s = torch.cuda.current_stream(x_local.device).cuda_stream
        xp, yp = x_local.data_ptr(), y_own.data_ptr()
        self.dev.spmv_tiles_ptr(xp, yp, self.t_lo, self.t_hi, s, f32=self.f32)
        for w in works:
            w.wait()
        if self.t_lo > 0:
            self.dev.spmv_tiles_ptr(xp, yp, 0, self.t_lo, s, f32=self.f32)
        if self.t_hi < self.n_tiles:
            self.dev.spmv_tiles_ptr(xp, yp, self.t_hi, self.n_tiles, s, f32=self.f32)
        return y_own

    @property
    def launches_per_step(self) -> int:
        return int(self.t_hi > self.t_lo) + int(self.t_lo > 0) + int(self.t_hi < self.n_tiles)

    def step_host(self, x_host, y_host, x_local, y_own, chunks: int = 8):
        """One SpMV from this rank's pinned host x slice to its pinned host y
        slice, overlapped like the single-GPU pipeline (csrk_spmv_host): x
        goes up in plane-aligned chunks (the two boundary chunks first, so
        the halo exchange starts early), each chunk's interior tiles run as
        soon as the x chunks they read have landed, the boundary tiles after
        the exchange, and y goes down per chunk on a third stream."""
        import torch

        lay, p = self.lay, self.lay.plane
        if self._pipe is None or self._pipe[0] != chunks:
            planes = lay.z1 - lay.z0
            k = max(1, min(chunks, planes))
            rcut = [lay.plane * (planes * c // k) for c in range(k + 1)]
            tr = np.asarray(self.dev.tile_rows(), dtype=np.int64)
            tcut = [min(max(int(np.searchsorted(tr, r, side="left")), self.t_lo), self.t_hi)
                    for r in rcut]
            tcut[0], tcut[-1] = self.t_lo, self.t_hi
            self._pipe = (chunks, k, rcut, tcut, tr, torch.cuda.Stream(), torch.cuda.Stream())
        _, k, rcut, tcut, tr, h2d, d2h = self._pipe
        cur = torch.cuda.current_stream()
        own0 = lay.own_off
        ev_x = [torch.cuda.Event() for _ in range(k)]
        order = [0] + ([k - 1] if k > 1 else []) + list(range(1, k - 1))
        h2d.wait_stream(cur)
        with torch.cuda.stream(h2d):
            for c in order:
                a, b = rcut[c], rcut[c + 1]
                x_local[own0 + a:own0 + b].copy_(x_host[a:b], non_blocking=True)
                ev_x[c].record(h2d)
        works = []
        if lay.world > 1:
            cur.wait_event(ev_x[0])
            cur.wait_event(ev_x[k - 1])
            works = self.exchange.start(x_local)
        s = cur.cuda_stream
        xp, yp = x_local.data_ptr(), y_own.data_ptr()
        d2h.wait_stream(cur)
        for c in range(k):
            if tcut[c + 1] > tcut[c]:
                # the x chunks the chunk's rows read: its real row span (a
                # tile may run past rcut[c + 1]) widened by one plane each way
                ra, rb = int(tr[tcut[c]]) - p, int(tr[tcut[c + 1]]) + p
                for j in range(k):
                    if rcut[j] < rb and rcut[j + 1] > ra:
                        cur.wait_event(ev_x[j])
                self.dev.spmv_tiles_ptr(xp, yp, tcut[c], tcut[c + 1], s, f32=self.f32)
                ev = torch.cuda.Event()
                ev.record(cur)
                d2h.wait_event(ev)
                a, b = int(tr[tcut[c]]), int(tr[tcut[c + 1]])
                with torch.cuda.stream(d2h):
                    y_host[a:b].copy_(y_own[a:b], non_blocking=True)
        for w in works:
            w.wait()
        for t0, t1 in ((0, self.t_lo), (self.t_hi, self.n_tiles)):
            if t1 > t0:
                for j in range(k):
                    cur.wait_event(ev_x[j])
                self.dev.spmv_tiles_ptr(xp, yp, t0, t1, s, f32=self.f32)
                ev = torch.cuda.Event()
                ev.record(cur)
                d2h.wait_event(ev)
                a, b = int(tr[t0]), int(tr[t1])
                with torch.cuda.stream(d2h):
                    y_host[a:b].copy_(y_own[a:b], non_blocking=True)
        cur.wait_stream(d2h)
        return y_host


class DeviceCgSteps:
    """The device step kernels of csrc/cg.cu behind DistCG (raw pointers,
    the caller's current stream)."""

    RED_BLOCKS = 592  # csrc/cg.cu kRedBlocks

    def __init__(self, device):
        import torch

        self.sc = torch.zeros(8, dtype=torch.float64, device=device)
        self.part = torch.zeros(self.RED_BLOCKS, dtype=torch.float64, device=device)
        self.cnt = torch.zeros(4, dtype=torch.int32, device=device)

    @staticmethod
    def _args(t):
        import torch

        from . import _native as nat

        vt = nat.CSRK_F32 if t.dtype == torch.float32 else nat.CSRK_F64
        s = C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
        return vt, s

    def dot(self, a, b, slot: int):
        from . import _native as nat

        vt, s = self._args(a)
        nat.call("csrk_vec_dot", vt, a.numel(), C.c_void_p(a.data_ptr()),
                 C.c_void_p(b.data_ptr()), C.c_void_p(self.part.data_ptr()),
                 C.c_void_p(self.cnt.data_ptr()), C.c_void_p(self.sc.data_ptr() + 8 * slot), s)

    def update(self, x, r, p, ap):
        from . import _native as nat

        vt, s = self._args(x)
        nat.call("csrk_cg_update", vt, x.numel(), C.c_void_p(x.data_ptr()),
                 C.c_void_p(r.data_ptr()), C.c_void_p(p.data_ptr()), C.c_void_p(ap.data_ptr()),
                 C.c_void_p(self.sc.data_ptr()), C.c_void_p(self.part.data_ptr()),
                 C.c_void_p(self.cnt.data_ptr()), s)

    def direction(self, p, r):
        from . import _native as nat

        vt, s = self._args(p)
        nat.call("csrk_cg_direction", vt, p.numel(), C.c_void_p(p.data_ptr()),
                 C.c_void_p(r.data_ptr()), C.c_void_p(self.sc.data_ptr()),
                 C.c_void_p(self.cnt.data_ptr()), s)


class DistCG:
    """Conjugate gradients on a partitioned operator (BASELINE config C4:
    repeated SpMVs as a CG inner loop, at N GPUs).

    ``op`` is a SlabSpMV or a DistSpMV: ``.own`` (the owned slice of its
    local x), ``.n_local_cols``, ``.n_own`` and ``.step(x_local, y_own)``
    (halo exchange overlapped with the interior tiles, then the boundary
    tiles).  The search direction lives in a local-x buffer so its halo can
    be exchanged; the other vectors are this rank's slices.  Per iteration:
    the SpMV, then the device step kernels of csrc/cg.cu (csrk_vec_dot,
    csrk_cg_update, csrk_cg_direction -- each finishes its reduction on the
    device) with one NCCL all-reduce of a device scalar after the first two:
    no host synchronisation, so :meth:`graphed` captures the whole run into
    one CUDA graph.  The recurrence is csrk_cg's (classic CG).  ``steps``
    replaces the step kernels (the CPU tests pass a host stand-in)."""

    def __init__(self, op, group=None, steps=None):
        import torch.distributed as dist

        self.op, self.group = op, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self._steps = steps

    def _allreduce(self, t):
        import torch.distributed as dist

        if self.world > 1:
            dist.all_reduce(t, group=self.group)

    def scratch(self, b_own):
        import torch

        return (torch.zeros(self.op.n_local_cols, dtype=b_own.dtype, device=b_own.device),
                torch.empty_like(b_own), torch.empty_like(b_own))

    def run(self, b_own, x_own, iters: int, scratch=None):
        """``iters`` CG iterations from x_own (updated in place); returns
        (x_own, rr) with rr the device scalar of the last r.r."""
        import torch

        op = self.op
        if self._steps is None:
            self._steps = DeviceCgSteps(b_own.device)
        st = self._steps
        sc = st.sc
        p_local, r, ap = scratch if scratch is not None else self.scratch(b_own)
        p = p_local[op.own]
        p.copy_(x_own)
        op.step(p_local, ap)  # ap = A x0
        torch.sub(b_own, ap, out=r)
        p.copy_(r)
        st.dot(r, r, 0)
        self._allreduce(sc[0:1])
        for _ in range(iters):
            op.step(p_local, ap)
            st.dot(p, ap, 1)
            self._allreduce(sc[1:2])
            st.update(x_own, r, p, ap)
            self._allreduce(sc[2:3])
            st.direction(p, r)
        return x_own, sc[0:1]

    def graphed(self, b_own, x_own, iters: int, scratch=None):
        """The whole run (x_own reset to 0, the initial residual, ``iters``
        iterations) captured once into a CUDA graph -- SpMV launches, halo
        point-to-point, all-reduces and step kernels; returns the graph
        (``.replay()``)."""
        import torch

        scratch = scratch if scratch is not None else self.scratch(b_own)
        s = torch.cuda.Stream(device=b_own.device)
        s.wait_stream(torch.cuda.current_stream(b_own.device))
        with torch.cuda.stream(s):  # warm-up outside the capture (plans, comms)
            x_own.zero_()
            self.run(b_own, x_own, iters, scratch)
        torch.cuda.current_stream(b_own.device).wait_stream(s)
        torch.cuda.synchronize(b_own.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            x_own.zero_()
            self.run(b_own, x_own, iters, scratch)
        return g

    def launches_per_iteration(self) -> int:
        return self.op.launches_per_step + 3


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


def local_block(m, r0: int, r1: int, col0: int = 0) -> RankBlock:
    """Slice a CsrKMatrix (k = 3) at SSR-aligned rows [r0, r1); columns are
    shifted by ``-col0`` (the first global column of the rank's local x)."""
    b = m.base
    rp = b.row_ptr.astype(np.int64)
    p0, p1 = int(rp[r0]), int(rp[r1])
    sr = m.sr_ptr.astype(np.int64)
    ssr = m.ssr_ptr.astype(np.int64)
    s0, s1 = int(np.searchsorted(sr, r0)), int(np.searchsorted(sr, r1))
    q0, q1 = int(np.searchsorted(ssr, s0)), int(np.searchsorted(ssr, s1))
    if sr[s0] != r0 or sr[s1] != r1 or ssr[q0] != s0 or ssr[q1] != s1:
        raise ValueError("rank block must start and end on super-super-row boundaries")
    ci = b.col_idx[p0:p1]
    if col0:
        ci = (ci.astype(np.int64) - col0).astype(np.uint32)
    return RankBlock(
        r0=r0, r1=r1, n_cols=b.n_cols - col0,
        row_ptr=(rp[r0:r1 + 1] - p0).astype(np.uint32),
        col_idx=ci, vals=b.vals[p0:p1],
        sr_ptr=(sr[s0:s1 + 1] - r0).astype(np.uint32),
        ssr_ptr=(ssr[q0:q1 + 1] - s0).astype(np.uint32))


def interior_rows(row_ptr, col_idx, own0: int, own1: int) -> tuple:
    """[a, b): a row range of a block whose every row reads only columns in
    [own0, own1) -- rows are sorted by column, so a row's first / last entry
    are its extremes.  Rows before ``a`` or from ``b`` on may read halo
    columns (the block's first and last rows under a banded order)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int64)
    n = rp.shape[0] - 1
    nz = rp[1:] > rp[:-1]
    first = np.where(nz, ci[np.minimum(rp[:-1], max(len(ci) - 1, 0))], own0)
    last = np.where(nz, ci[np.maximum(rp[1:] - 1, 0)], own0)
    lo_bad = np.flatnonzero(nz & (first < own0))
    hi_bad = np.flatnonzero(nz & (last >= own1))
    a = int(lo_bad[-1]) + 1 if lo_bad.size else 0
    b = int(hi_bad[0]) if hi_bad.size else n
    return a, max(a, b)


class XExchange:
    """Fills the halo of one rank's local x (global columns [x0, x1), owned
    slice [r0, r1) inside it) from the peers that own those columns.

      "halo"       (default) one ``batch_isend_irecv`` of exactly the
                   contiguous windows each rank's rows read from each peer
                   (halo_plan); with Band-k ordering these are narrow bands
                   next to the owned slice;
      "allgather"  the literal north-star collective: every rank's owned
                   slice, padded to the largest, all-gathered into one
                   buffer, then the footprint windows copied into place.

    Both post asynchronously (``start``) and return works the caller waits
    on (``finish``) -- the interior rows are computed in between.  Works on
    CPU tensors over gloo (tests) and CUDA tensors over NCCL."""

    def __init__(self, rank: int, world: int, cuts, fps, x0: int, mode: str = "halo",
                 group=None):
        if mode not in ("halo", "allgather"):
            raise ValueError(f"unknown exchange mode {mode!r}")
        self.rank, self.world, self.mode, self.group = rank, world, mode, group
        self.cuts = [int(c) for c in cuts]
        self.x0 = int(x0)
        plan = halo_plan(self.cuts, fps)
        self.sends = [(d, a, b) for s, d, a, b in plan if s == rank]
        self.recvs = [(s, a, b) for s, d, a, b in plan if d == rank]
        self.maxlen = max(self.cuts[g + 1] - self.cuts[g] for g in range(world))
        self._bufs = None
        self._pending = []

    def bytes_received(self, itemsize: int = 8) -> int:
        if self.mode == "allgather":
            return (self.world - 1) * self.maxlen * itemsize
        return sum(b - a for _, a, b in self.recvs) * itemsize

    def bytes_sent(self, itemsize: int = 8) -> int:
        if self.mode == "allgather":
            return self.maxlen * itemsize
        return sum(b - a for _, a, b in self.sends) * itemsize

    def start(self, x_local) -> list:
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return []
        x0 = self.x0
        if self.mode == "halo":
            ops = [dist.P2POp(dist.isend, x_local[a - x0:b - x0], d, group=self.group)
                   for d, a, b in self.sends]
            ops += [dist.P2POp(dist.irecv, x_local[a - x0:b - x0], s, group=self.group)
                    for s, a, b in self.recvs]
            # a rank without peers posts nothing; the communicator already
            # exists (the constructor's collective), so the other ranks'
            # batches do not wait on it
            self._pending = []
            return dist.batch_isend_irecv(ops) if ops else []
        if self._bufs is None or self._bufs[0].device != x_local.device or \
                self._bufs[0].dtype != x_local.dtype:
            self._bufs = (torch.zeros(self.maxlen, dtype=x_local.dtype, device=x_local.device),
                          torch.zeros(self.world * self.maxlen, dtype=x_local.dtype,
                                      device=x_local.device))
        mine, every = self._bufs
        lo, hi = self.cuts[self.rank], self.cuts[self.rank + 1]
        mine[:hi - lo].copy_(x_local[lo - x0:hi - x0])
        work = dist.all_gather_into_tensor(every, mine, group=self.group, async_op=True)
        self._pending = [(s, a, b) for s, a, b in self.recvs]
        return [work]

    def finish(self, x_local, works) -> None:
        for w in works:
            w.wait()
        if self.mode == "allgather":
            _, every = self._bufs
            for s, a, b in self._pending:
                off = s * self.maxlen + (a - self.cuts[s])
                x_local[a - self.x0:b - self.x0].copy_(every[off:off + (b - a)])

    def __call__(self, x_local):
        self.finish(x_local, self.start(x_local))
        return x_local


class DistSpMV:
    """y_own = A[r0:r1, :] x on this rank's GPU.

    The packed matrix's super-super-rows are split by nonzeros
    (partition_by_nnz, the reference's static chunks kernels.py:150-155 with
    nonzero weights).  The rank keeps only its rows, with columns local to
    its footprint: x_local holds global columns [x0, x1) -- the owned slice
    [r0, r1) plus the halo its rows read -- never a global-length x.

    One step posts the exchange of the halo, runs the interior tiles (rows
    that read owned columns only; interior_rows) while it is in flight,
    waits, then runs the boundary tiles before / after them: the NVLink
    transfer overlaps the bulk of the SpMV.  y is bitwise the single-GPU
    result (rows are summed whole, in the reference's order)."""

    def __init__(self, m, rank: int, world: int, mode: str = "halo", group=None,
                 device=None, f32: bool = False, variant: str = "serial", nx: int = 1):
        from . import _native as nat

        b = m.base
        self.cuts = partition_by_nnz(b.row_ptr, m.sr_ptr, m.ssr_ptr, world)
        self.fps = footprints(b.row_ptr, b.col_idx, self.cuts)
        self.rank, self.world = rank, world
        self.r0, self.r1 = int(self.cuts[rank]), int(self.cuts[rank + 1])
        lo, hi = (int(v) for v in self.fps[rank])
        self.x0 = min(lo, self.r0) if hi > lo else self.r0
        self.x1 = max(hi, self.r1) if hi > lo else self.r1
        blk = local_block(m, self.r0, self.r1, col0=self.x0)
        self.n_own = self.r1 - self.r0
        self.n_local_cols = self.x1 - self.x0
        self.nnz_local = int(blk.row_ptr[-1])
        self.nnz_total = b.nnz
        self.n = b.n_rows
        self.f32 = f32
        self.var = nat.CSRK_STRIDED if variant == "strided" else nat.CSRK_SERIAL
        self.nx = int(nx) if variant == "strided" else 1
        self.dev = None
        self.t_lo = self.t_hi = self.n_tiles = 0
        if self.n_own > 0:
            self.dev = nat.DeviceMatrix.upload(
                blk.row_ptr, blk.col_idx, blk.vals, self.n_own, self.n_local_cols, k=3,
                sr_ptr=blk.sr_ptr, ssr_ptr=blk.ssr_ptr, device=device, f32=f32)
            self.dev.prepare(self.var, self.nx, f32)
            self.n_tiles = self.dev.plan()["n_tiles"]
            a, bb = interior_rows(blk.row_ptr, blk.col_idx, self.r0 - self.x0,
                                  self.r1 - self.x0)
            self.t_lo, self.t_hi = interior_tiles(self.dev.tile_rows(), a, bb)
        self.exchange = XExchange(rank, world, self.cuts, self.fps, self.x0, mode, group)
        _collective_warmup(group)

    @property
    def own(self) -> slice:
        """The owned x entries inside x_local."""
        return slice(self.r0 - self.x0, self.r1 - self.x0)

    def new_x_local(self, dtype=None, device=None):
        import torch

        dtype = dtype or (torch.float32 if self.f32 else torch.float64)
        return torch.zeros(max(1, self.n_local_cols), dtype=dtype, device=device or "cuda")

    def _tiles(self, x_local, y_own, t0, t1, s):
        if t1 > t0:
            self.dev.spmv_tiles_ptr(x_local.data_ptr(), y_own.data_ptr(), t0, t1, s,
                                    variant=self.var, nx=self.nx, f32=self.f32)

    def step(self, x_local, y_own):
        """Post the x exchange, interior tiles, wait, boundary tiles -- all
        ordered on the current stream (NCCL's works wait on it and it waits
        on them)."""
        import torch

        works = self.exchange.start(x_local)
        if self.dev is not None:
            s = torch.cuda.current_stream(x_local.device).cuda_stream
            self._tiles(x_local, y_own, self.t_lo, self.t_hi, s)
            self.exchange.finish(x_local, works)
            self._tiles(x_local, y_own, 0, self.t_lo, s)
            self._tiles(x_local, y_own, self.t_hi, self.n_tiles, s)
        else:
            self.exchange.finish(x_local, works)
        return y_own

    @property
    def launches_per_step(self) -> int:
        if self.dev is None:
            return 0
        n_long = 1 if self.dev.plan()["n_long"] > 0 else 0
        parts = [self.t_hi > self.t_lo, self.t_lo > 0, self.t_hi < self.n_tiles]
        return sum(parts) * (1 + n_long)

    def local_bytes(self, itemsize: int) -> int:
        """Algorithmic HBM bytes of this rank's SpMV (SURVEY.md §8(d) on the
        rank's block: its nonzeros, row pointers, local x and y)."""
        return (self.nnz_local * (itemsize + 4) + 4 * (self.n_own + 1)
                + (self.n_local_cols + self.n_own) * itemsize)


def native_partition(m, parts: int) -> np.ndarray:
    """partition_by_nnz through the C-ABI (csrk_mg_partition)."""
    from . import _native as nat

    rp = np.ascontiguousarray(m.base.row_ptr, dtype=np.uint32)
    sp = np.ascontiguousarray(m.sr_ptr, dtype=np.uint32)
    ssp = np.ascontiguousarray(m.ssr_ptr, dtype=np.uint32)
    cuts = np.zeros(parts + 1, dtype=np.int64)
    nat.call("csrk_mg_partition", nat.u32p(rp), nat.u32p(sp), nat.u32p(ssp), len(ssp) - 1,
             parts, nat.i64p(cuts))
    return cuts


def native_footprints(row_ptr, col_idx, cuts) -> np.ndarray:
    """footprints through the C-ABI (csrk_mg_footprints)."""
    from . import _native as nat

    rp = np.ascontiguousarray(row_ptr, dtype=np.uint32)
    ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
    cu = np.ascontiguousarray(cuts, dtype=np.int64)
    fps = np.zeros((len(cu) - 1, 2), dtype=np.int64)
    nat.call("csrk_mg_footprints", nat.u32p(rp), nat.u32p(ci), nat.i64p(cu), len(cu) - 1,
             nat.i64p(fps))
    return fps


def native_halo_plan(cuts, fps) -> list:
    """halo_plan through the C-ABI (csrk_mg_plan)."""
    import ctypes as C

    from . import _native as nat

    cu = np.ascontiguousarray(cuts, dtype=np.int64)
    fp = np.ascontiguousarray(fps, dtype=np.int64)
    count = C.c_int64()
    nat.call("csrk_mg_plan", len(cu) - 1, nat.i64p(cu), nat.i64p(fp), None, 0, C.byref(count))
    out = np.zeros((max(count.value, 1), 4), dtype=np.int64)
    nat.call("csrk_mg_plan", len(cu) - 1, nat.i64p(cu), nat.i64p(fp), nat.i64p(out),
             count.value, C.byref(count))
    return [tuple(int(v) for v in row) for row in out[:count.value]]


class NativeDistSpMV:
    """DistSpMV behind the C-ABI (csrk_mg_create / csrk_mg_spmv, SURVEY.md
    §8(b)): the same nnz-balanced SSR blocks, footprint-local x and halo /
    all-gather exchange, with NCCL driven from the library (its own
    communicator, created from a unique id rank 0 broadcasts over the
    torch.distributed group) and the interior / boundary tile split done in
    C++.  y_own is bitwise the single-GPU y."""

    def __init__(self, m, rank: int, world: int, mode: str = "halo", group=None,
                 device=None, f32: bool = False, variant: str = "serial", nx: int = 1,
                 communicator: bool = True):
        """communicator=False: no NCCL communicator; the caller fills the
        halo of x_local itself before step() (tests on one GPU)."""
        import ctypes as C

        import torch

        from . import _native as nat

        if mode not in ("halo", "allgather"):
            raise ValueError(f"unknown exchange mode {mode!r}")
        b = m.base
        self.cuts = native_partition(m, world)
        self.fps = native_footprints(b.row_ptr, b.col_idx, self.cuts)
        self.rank, self.world, self.f32 = rank, world, f32
        self.r0, self.r1 = int(self.cuts[rank]), int(self.cuts[rank + 1])
        lo, hi = (int(v) for v in self.fps[rank])
        self.x0 = min(lo, self.r0) if hi > lo else self.r0
        self.x1 = max(hi, self.r1) if hi > lo else self.r1
        self.n_own = self.r1 - self.r0
        self.n_local_cols = self.x1 - self.x0
        self.var = nat.CSRK_STRIDED if variant == "strided" else nat.CSRK_SERIAL
        self.nx = int(nx) if variant == "strided" else 1
        self.dev = None
        self.nnz_local = 0
        if self.n_own > 0:
            blk = local_block(m, self.r0, self.r1, col0=self.x0)
            self.nnz_local = int(blk.row_ptr[-1])
            self.dev = nat.DeviceMatrix.upload(
                blk.row_ptr, blk.col_idx, blk.vals, self.n_own, self.n_local_cols, k=3,
                sr_ptr=blk.sr_ptr, ssr_ptr=blk.ssr_ptr, device=device, f32=f32)
            self.dev.prepare(self.var, self.nx, f32)
        uid = C.create_string_buffer(nat.CSRK_MG_ID_BYTES)
        if communicator and rank == 0:
            nat.call("csrk_mg_unique_id", uid)
        if communicator and world > 1:
            import torch.distributed as dist

            on = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
            t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).to(on)
            dist.broadcast(t, src=0, group=group)
            uid = C.create_string_buffer(bytes(t.cpu().numpy().tobytes()),
                                         nat.CSRK_MG_ID_BYTES)
        self._cuts_c = np.ascontiguousarray(self.cuts, dtype=np.int64)
        self._fps_c = np.ascontiguousarray(self.fps, dtype=np.int64)
        out = C.c_void_p()
        nat.call("csrk_mg_create", rank, world, uid if communicator else None,
                 nat.i64p(self._cuts_c),
                 nat.i64p(self._fps_c), self.dev.ptr if self.dev is not None else None,
                 self.x0, nat.CSRK_MG_ALLGATHER if mode == "allgather" else nat.CSRK_MG_HALO,
                 C.byref(out))
        self.ptr = out

    @property
    def own(self) -> slice:
        return slice(self.r0 - self.x0, self.r1 - self.x0)

    def new_x_local(self, dtype=None, device=None):
        import torch

        dtype = dtype or (torch.float32 if self.f32 else torch.float64)
        return torch.zeros(max(1, self.n_local_cols), dtype=dtype, device=device or "cuda")

    def info(self) -> dict:
        from . import _native as nat

        out = np.zeros(9, dtype=np.int64)
        nat.call("csrk_mg_info", self.ptr, nat.i64p(out))
        keys = ("interior_a", "interior_b", "t_lo", "t_hi", "n_tiles", "sent", "received",
                "n_sends", "n_recvs")
        return dict(zip(keys, (int(v) for v in out)))

    @property
    def exchange(self):
        """bytes_received / bytes_sent per step, like XExchange."""
        info = self.info()

        class _Bytes:
            @staticmethod
            def bytes_received(itemsize: int = 8) -> int:
                return info["received"] * itemsize

            @staticmethod
            def bytes_sent(itemsize: int = 8) -> int:
                return info["sent"] * itemsize
        return _Bytes

    @property
    def launches_per_step(self) -> int:
        if self.dev is None:
            return 0
        i = self.info()
        if i["n_tiles"] < 0:  # plan not read yet (before the first step)
            i["t_lo"], i["t_hi"], i["n_tiles"] = 0, 1, 1
        n_long = 1 if self.dev.plan()["n_long"] > 0 else 0
        parts = [i["t_hi"] > i["t_lo"], i["t_lo"] > 0, i["t_hi"] < i["n_tiles"]]
        return sum(parts) * (1 + n_long)

    def local_bytes(self, itemsize: int) -> int:
        return (self.nnz_local * (itemsize + 4) + 4 * (self.n_own + 1)
                + (self.n_local_cols + self.n_own) * itemsize)

    def step(self, x_local, y_own):
        import torch

        from . import _native as nat

        s = torch.cuda.current_stream(x_local.device).cuda_stream
        nat.call("csrk_mg_spmv", self.ptr, nat.CSRK_F32 if self.f32 else nat.CSRK_F64,
                 self.var, self.nx, x_local.data_ptr(),
                 y_own.data_ptr() if y_own is not None and y_own.numel() else None, s)
        return y_own

    def close(self):
        from . import _native as nat

        if getattr(self, "ptr", None) is not None and self.ptr.value:
            nat.call("csrk_mg_destroy", self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _collective_warmup(group=None) -> None:
    """One collective over the group before any point-to-point batch: with
    NCCL the first batch_isend_irecv must otherwise involve every rank, and
    a rank with no halo posts none (torch's batch_isend_irecv contract)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.zeros(1, device=dev)
    dist.all_reduce(t, group=group)


# kept for callers of the round-1 name: the exchange on a full-length x
def Exchange(rank, world, cuts, fps, mode="halo", group=None):  # noqa: N802
    return XExchange(rank, world, cuts, fps, 0, mode, group)


METRIC = "SpMV GFLOP/s and achieved HBM GB/s (% of peak) at 1/2/4/8 B200 vs host CPU"


def _max_over_ranks(v: float) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _min_over_ranks(v: int) -> int:
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(v)], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item())


def _sum_over_ranks(v: int) -> int:
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(v)], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def bench_slabs(args, log, rank: int, world: int, local: int, sampler=None, peak=None,
                side: int = 256):
    """Weak scaling: every rank owns a C2-sized slab (side^3 rows: side planes
    of side x side) of the 3D 7-point Laplacian on a side x side x
    (side * world) grid, generated in its own HBM; one step = one SpMV of the
    global matrix (halo planes over NCCL overlapped with the interior tiles).
    Device time with CUDA events, max over ranks; e2e adds the H2D of each
    rank's x slice and the D2H of its y slice from / to pinned host memory."""
    import time

    import torch
    import torch.distributed as dist

    from .bench import spmv_bytes

    shape = (side * world, side, side)
    dtype = torch.float32 if args.fp32 else torch.float64
    vb = 4 if args.fp32 else 8
    op = SlabSpMV(shape, 7, rank, world, device=local, f32=args.fp32)
    lay = op.lay
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x_local = torch.zeros(lay.n_cols, dtype=dtype, device="cuda")
    own = slice(lay.own_off, lay.own_off + lay.n_own)
    x_local[own] = (torch.rand(lay.n_own, generator=gen, device="cuda",
                               dtype=torch.float64) * 2 - 1).to(dtype)
    y = torch.empty(lay.n_own, dtype=dtype, device="cuda")

    def step():
        op.step(x_local, y)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    # untimed load under the clock sampler: the same step count on every
    # rank (point-to-point exchanges must pair up), ~0.5 s
    t0 = time.perf_counter()
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    est = _max_over_ranks((time.perf_counter() - t0) / 5)
    burn = max(5, int(0.5 / max(est, 1e-6)))

    class _Null:
        def __enter__(self):
            return self

        def __exit__(self, *a):
            return False

        def summary(self):
            return None

    clk_ctx = sampler(torch.cuda.current_device()) if (sampler and rank == 0) else _Null()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with clk_ctx as clk:
        for _ in range(burn):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = _max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    nnz_total = _sum_over_ranks(op.nnz_local)
    rows_total = _sum_over_ranks(lay.n_own)

    # e2e: public API per rank with host buffers (x slice up, y slice down)
    x_pin = torch.empty(lay.n_own, dtype=dtype, pin_memory=True)
    x_pin.copy_(x_local[own])
    y_pin = torch.empty(lay.n_own, dtype=dtype, pin_memory=True)
    e2e_steps = max(3, min(args.steps, 20))
    for it in range(e2e_steps + 1):
        if it == 1:
            torch.cuda.synchronize()
            dist.barrier()
            te = time.perf_counter()
        op.step_host(x_pin, y_pin, x_local, y)
        torch.cuda.synchronize()
    e2e_s = _max_over_ranks((time.perf_counter() - te) / e2e_steps)
    if rank != 0:
        return None
    algo = spmv_bytes(lay.n_own, lay.n_cols, op.nnz_local, vb)
    gbs = algo / (ms * 1e-3) / 1e9
    peak_v, peak_src = peak if peak else (None, None)
    return {
        "metric": METRIC,
        "value": round(2.0 * nnz_total / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.fp32 else "f64",
        "data": "synthetic (3D 7-point Laplacian generated in HBM per rank, "
                "x ~ U[-1,1) per rank)",
        "config": {"workload": f"C2-sized slab per GPU: 3D 7-point Laplacian "
                               f"{side}x{side}x{side * world} ({side}^3 rows per rank), "
                               "natural order, CSR-k k=3 uniform SR 8 / SSR 8",
                   "n_rows": rows_total, "nnz": nnz_total,
                   "parallelism": f"z-slab row blocks x{world}, NCCL halo planes "
                                  "overlapped with the interior tiles",
                   "halo_bytes_per_rank": op.exchange.bytes_received(vb),
                   "l2": "inputs larger than L2; no flush"},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak_v,
                     "unit": "GB/s", "frac": round(gbs / peak_v, 4) if peak_v else None,
                     "peak_source": peak_src, "per": "rank 0's GPU (its slab's "
                     "algorithmic bytes / the max-over-ranks step time)",
                     "traffic": None, "algorithmic_bytes_per_launch": algo},
        "e2e": {"value": round(2.0 * nnz_total / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": lay.n_own * vb * world,
                "d2h_bytes_per_step": lay.n_own * vb * world,
                "ms_per_step": round(e2e_s * 1e3, 3),
                "call": "dist.SlabSpMV.step_host with pinned host x / y slices per rank "
                        "(chunked H2D, halo exchange, interior / boundary tiles, D2H)"},
        "cpu_baseline": None,
        "gpu_launches": args.steps * op.launches_per_step,
        "clocks": clk.summary() if clk is not None else None,
    }


def bench_cg_slabs(args, log, rank: int, world: int, local: int, sampler=None, peak=None):
    """C4 at N GPUs (strong scaling): the side^3 7-point Laplacian split into
    z-slabs, ``args.iters`` CG iterations per step (DistCG: halo planes +
    interior/boundary SpMV + two all-reduced dots per iteration)."""
    import time

    import torch
    import torch.distributed as dist

    from .bench import spmv_bytes

    side = args.side
    shape = (side, side, side)
    dtype = torch.float32 if args.fp32 else torch.float64
    vb = 4 if args.fp32 else 8
    op = SlabSpMV(shape, 7, rank, world, device=local, f32=args.fp32)
    lay = op.lay
    solver = DistCG(op)
    gen = torch.Generator(device="cuda").manual_seed(2000 + rank)
    b = (torch.rand(lay.n_own, generator=gen, device="cuda", dtype=torch.float64) * 2
         - 1).to(dtype)
    x = torch.zeros_like(b)
    scratch = (torch.zeros(lay.n_cols, dtype=dtype, device="cuda"), torch.empty_like(b),
               torch.empty_like(b))
    iters = args.iters

    def eager_step():
        x.zero_()
        solver.run(b, x, iters, scratch=scratch)

    for _ in range(max(3, args.warmup)):
        eager_step()
    torch.cuda.synchronize()
    # one step = one replay of the whole run captured as a CUDA graph (SpMV
    # launches, halo point-to-point, all-reduces and step kernels): the host
    # enqueues ~10 operations per iteration, which at N = 8 (0.5 ms of GPU
    # work per iteration) it could otherwise only just keep ahead of
    graph = None
    if getattr(args, "graph", True):
        try:
            graph = solver.graphed(b, x, iters, scratch=scratch)
            graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:
            log(f"[bench] CUDA graph capture of the distributed CG failed ({exc}); eager")
            graph = None
            torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            eager_step()

    dist.barrier()
    clk_ctx = sampler(torch.cuda.current_device()) if (sampler and rank == 0) else None
    if clk_ctx is not None:
        clk_ctx.__enter__()
    step()
    torch.cuda.synchronize()
    dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    if clk_ctx is not None:
        clk_ctx.__exit__(None, None, None)
    ms = _max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    nnz_total = _sum_over_ranks(op.nnz_local)
    b_pin = torch.empty(lay.n_own, dtype=dtype, pin_memory=True)
    b_pin.copy_(b)
    x_pin = torch.empty(lay.n_own, dtype=dtype, pin_memory=True)
    torch.cuda.synchronize()
    dist.barrier()
    te = time.perf_counter()
    e2e_steps = 2
    for _ in range(e2e_steps):
        b.copy_(b_pin, non_blocking=True)
        step()
        x_pin.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = _max_over_ranks((time.perf_counter() - te) / e2e_steps)
    if rank != 0:
        return None
    flops = 2.0 * nnz_total * iters
    it_bytes = spmv_bytes(lay.n_own, lay.n_cols, op.nnz_local, vb) + 11 * lay.n_own * vb
    gbs = it_bytes * iters / (ms * 1e-3) / 1e9
    peak_v, peak_src = peak if peak else (None, None)
    return {
        "metric": METRIC, "value": round(flops / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if args.fp32 else "f64",
        "data": "synthetic (7-point Laplacian slabs generated in HBM, b ~ U[-1,1))",
        "config": {"workload": f"C4: {iters} SpMVs as a CG inner loop on the {side}^3 "
                               f"7-point Laplacian, z-slabs over {world} GPUs",
                   "config_id": "C4", "nnz": nnz_total, "iterations_per_step": iters,
                   "parallelism": f"z-slab row blocks x{world}, NCCL halo planes + "
                                  "2 all-reduces per iteration",
                   "ms_per_iteration": round(ms / iters, 5)},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak_v, "unit": "GB/s",
                     "frac": round(gbs / peak_v, 4) if peak_v else None,
                     "peak_source": peak_src, "per": "rank 0's GPU", "traffic": None,
                     "algorithmic_bytes_per_iteration": int(it_bytes)},
        "e2e": {"value": round(flops / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": lay.n_own * vb * world,
                "d2h_bytes_per_step": lay.n_own * vb * world,
                "ms_per_step": round(e2e_s * 1e3, 3), "call": "dist.DistCG.run per rank"},
        "cpu_baseline": None,
        "gpu_launches": args.steps * iters * solver.launches_per_iteration(),
        "timed_as": "one CUDA graph per step" if graph is not None else "eager steps",
        "clocks": clk_ctx.summary() if clk_ctx is not None else None,
    }


def bench_blocks(args, log, rank: int, world: int, local: int, sampler=None, peak=None,
                 oracle_check=None):
    """Strong scaling of one config's CSR-k matrix (the N = 1 bench line's
    matrix: synthetic input, native Band-k with the B200 model's sizes, device
    pack) over ``world`` GPUs: super-super-rows split by nonzeros
    (DistSpMV), x halo over NCCL overlapped with the interior tiles.  Every
    rank builds the matrix on its own GPU (device Band-k is deterministic and
    bit-exact, ~2 s at C2), keeps its row block, and rank 0 also times the
    whole matrix on one GPU (T1) for the efficiency T1 / (N T_N).  Device
    time with CUDA events on the launching stream, max over ranks."""
    import time

    import torch
    import torch.distributed as dist

    import bench as _bench  # the driver script's builder (repo root)

    from .bench import spmv_bytes

    a, m, xp, params, build_t = _bench.build_matrix(args.config, log)
    n, nnz = a.n_rows, a.nnz
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    nx = params.block_dims.x if variant == "strided" else 1
    f32 = args.fp32
    dtype = torch.float32 if f32 else torch.float64
    vb = 4 if f32 else 8
    mode = getattr(args, "exchange", None) or os.environ.get("CSRK_EXCHANGE", "halo")
    native = getattr(args, "mg", "torch") == "native"
    cls = NativeDistSpMV if native else DistSpMV
    op = cls(m, rank, world, mode=mode, device=local, f32=f32, variant=variant, nx=nx)
    x_local = op.new_x_local(dtype)
    x_local[op.own] = torch.from_numpy(xp[op.r0:op.r1]).to("cuda", dtype)
    # columns outside the owned slice are the exchange's job: poison them
    # so a missing halo shows up in the parity check
    if op.own.start > 0:
        x_local[:op.own.start] = float("nan")
    if op.own.stop < x_local.numel():
        x_local[op.own.stop:] = float("nan")
    y = torch.empty(max(1, op.n_own), dtype=dtype, device="cuda")

    def step():
        op.step(x_local, y)

    # T1: the whole matrix on rank 0's GPU alone (the others wait)
    t1_ms = None
    if rank == 0:
        from . import kernels

        xf = torch.from_numpy(xp).to("cuda", dtype)
        yf = torch.empty(n, dtype=dtype, device="cuda")
        dims = params.block_dims

        def full():
            kernels.spmv_device(m, xf, yf, dims=dims, variant=variant)

        for _ in range(3):
            full()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(10, args.steps)
        e0.record()
        for _ in range(reps):
            full()
        e1.record()
        torch.cuda.synchronize()
        t1_ms = e0.elapsed_time(e1) / reps
        del xf, yf
    dist.barrier()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clk_ctx = sampler(torch.cuda.current_device()) if (sampler and rank == 0) else None
    if clk_ctx is not None:
        clk_ctx.__enter__()
    burn = max(5, args.warmup)
    for _ in range(burn):  # untimed load while the sampler collects
        step()
    torch.cuda.synchronize()
    if clk_ctx is not None:
        time.sleep(0.3)
    # host enqueue cost of one step (Python + NCCL + launches): at N = 8 a
    # C2 block takes ~35 us on the GPU, so a step that costs the host more
    # than that starves the device
    torch.cuda.synchronize()
    th = time.perf_counter()
    for _ in range(args.steps):
        step()
    host_us = (time.perf_counter() - th) / args.steps * 1e6
    torch.cuda.synchronize()
    # the C-ABI path: the K timed steps captured once into a CUDA graph
    # (NCCL send / recv, the interior / boundary launches and their events
    # are all stream-ordered), replayed in the timed region
    graph = None
    if native and getattr(args, "graph", True):
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(args.steps):
                    step()
            graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # capture unsupported here: time eager steps
            log(f"[bench] CUDA graph capture of the native steps failed ({exc}); eager steps")
            graph = None
            torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    if graph is not None:
        graph.replay()
    else:
        for _ in range(args.steps):
            step()
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    if clk_ctx is not None:
        clk_ctx.__exit__(None, None, None)
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    ms = _max_over_ranks(ms_rank)
    host_us = _max_over_ranks(host_us)
    # parity of this rank's rows against the oracle (the timed output)
    ok = True
    max_diff = 0.0
    if oracle_check is not None and op.n_own > 0:
        want = oracle_check(m, xp, variant, nx)[op.r0:op.r1]
        got = y[:op.n_own].double().cpu().numpy()
        if f32:
            from .kernels import host_row_sums

            b = m.base
            scale = host_row_sums(b.row_ptr, b.col_idx, np.abs(b.vals), np.abs(xp))[op.r0:op.r1]
            ok = bool(np.all(np.abs(got - want) <= 1e-5 * scale))
        else:
            ok = bool(np.array_equal(got, want))
        max_diff = float(np.max(np.abs(got - want))) if got.size else 0.0
    ok_all = _min_over_ranks(int(ok))
    # e2e: each rank's owned x slice up from pinned host memory, the step,
    # its y slice down; max over ranks
    x_pin = torch.empty(max(1, op.n_own), dtype=dtype, pin_memory=True)
    x_pin[:op.n_own] = x_local[op.own].cpu()
    y_pin = torch.empty(max(1, op.n_own), dtype=dtype, pin_memory=True)
    e2e_steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize()
    dist.barrier()
    te = 0.0
    for it in range(e2e_steps + 1):
        if it == 1:
            torch.cuda.synchronize()
            dist.barrier()
            te = time.perf_counter()
        x_local[op.own].copy_(x_pin[:op.n_own], non_blocking=True)
        op.step(x_local, y)
        y_pin[:op.n_own].copy_(y[:op.n_own], non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = _max_over_ranks((time.perf_counter() - te) / e2e_steps)
    ex_max = _max_over_ranks(op.exchange.bytes_received(vb))
    local_gbs = op.local_bytes(vb) / (ms_rank * 1e-3) / 1e9
    gbs_min = -_max_over_ranks(-local_gbs)
    launches = _sum_over_ranks(op.launches_per_step)
    if rank != 0:
        return None
    algo = spmv_bytes(n, n, nnz, vb)
    peak_v, peak_src = peak if peak else (None, None)
    gflops = 2.0 * nnz / (ms * 1e-3) / 1e9
    return {
        "metric": METRIC,
        "value": round(gflops, 2), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if f32 else "f64",
        "data": "synthetic (deterministic grid Laplacian / irregular rows, x ~ U[-1,1) seed 0)",
        "config": {"workload": _bench.CONFIG_TEXT.get(args.config, args.config),
                   "config_id": args.config, "n_rows": n, "nnz": nnz,
                   "ssrs_target": params.ssrs, "srs_target": params.srs,
                   "kernel": f"csrk_stream_kernel ({variant}"
                             + (f", nx={nx})" if variant == "strided" else ")"),
                   "parallelism": f"row blocks of whole super-super-rows x{world}, "
                                  f"balanced by nonzeros; {mode} x exchange over NCCL "
                                  "overlapped with the interior tiles"
                                  + ("; C-ABI csrk_mg_* (NCCL driven from the library)"
                                     if native else "; torch.distributed NCCL"),
                   "exchange_bytes_per_rank_max": ex_max,
                   "l2": "inputs larger than L2; no flush" if algo >= 4 * 126e6 / world
                         else "per-rank inputs may fit L2 at this N"},
        "hbm_gbs": round(algo / (ms * 1e-3) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(gbs_min, 1), "peak": peak_v,
                     "unit": "GB/s", "frac": round(gbs_min / peak_v, 4) if peak_v else None,
                     "peak_source": peak_src,
                     "per": "slowest rank: its block's algorithmic bytes / its own step time",
                     "traffic": None,
                     "algorithmic_bytes_per_launch": op.local_bytes(vb)},
        "t1_ms": round(t1_ms, 4) if t1_ms else None,
        "efficiency_t1_over_n_tn": round(t1_ms / (world * ms), 4) if t1_ms else None,
        "host_enqueue_us_per_step_max": round(host_us, 1),
        "timed_as": "one CUDA graph of the K steps" if graph is not None else "K eager steps",
        "parity": {"kind": "scaled 1e-5" if f32 else "bitwise", "ok": bool(ok_all),
                   "against": "oracle/csrk_oracle.c on the same CSR-k matrix and x",
                   "max_abs_diff_rank0": max_diff},
        "e2e": {"value": round(2.0 * nnz / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": n * vb, "d2h_bytes_per_step": n * vb,
                "ms_per_step": round(e2e_s * 1e3, 3),
                "call": f"dist.{cls.__name__}.step per rank with its pinned host x / y "
                        "slices" + (" (C-ABI csrk_mg_spmv)" if native else "")},
        "cpu_baseline": None,
        "gpu_launches": args.steps * launches,
        "clocks": clk_ctx.summary() if clk_ctx is not None else None,
        "build_seconds": {k: round(v, 2) for k, v in build_t.items()},
    }


def bench_main(args, log, sampler=None, peak=None, oracle_check=None):
    """bench.py --gpus N (one process per GPU, torchrun).  C1/C2/C3/C5: the
    config's CSR-k matrix split over the ranks (strong scaling, the same
    matrix and kernel as the N = 1 line; bench_blocks).  C4: the CG loop of
    the 512^3 Laplacian on z-slabs (strong scaling, bench_cg_slabs).
    ``--partition slab`` keeps round 1's weak-scaling slab run of C2."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    from . import _native as nat
    nat.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.config == "C4":
            return bench_cg_slabs(args, log, rank, world, local, sampler, peak)
        if getattr(args, "partition", "blocks") == "slab":
            return bench_slabs(args, log, rank, world, local, sampler, peak)
        return bench_blocks(args, log, rank, world, local, sampler, peak, oracle_check)
    finally:
        dist.destroy_process_group()
