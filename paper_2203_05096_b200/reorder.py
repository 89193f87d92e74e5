"""Band-k reordering and super-row derivation, native.

Drop-in for the reference's ``csrk.reorder`` (pkg/src/csrk/reorder.py).  All
graph work runs in libcsrk_cuda.so, in two bit-identical implementations that
reproduce every greedy tie-break of the reference (pinned by tests/golden,
including the full-size C2 / C3 / C5 digests):

  device  csrc/{graph,rcm,coarsen,bandk_dev}.cu -- radix-sort graph building,
          level-synchronous exact Cuthill-McKee, Jacobi fixed-point matching
          and block expansion (the default when a GPU is present);
  host    csrc/bandk.cpp -- the sequential restatement (OpenMP where rows are
          independent), used without a GPU and for the graph-level helpers.

The Python layer only converts between the reference's array-holding objects
and the C-ABI.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .format import CsrMatrix, Permutation

__all__ = [
    "AdjacencyGraph",
    "CoarseningMap",
    "BandKResult",
    "build_graph",
    "heavy_edge_matching",
    "coarsen",
    "weighted_bandwidth_order",
    "band_k",
    "MIN_MATCH_SHRINK",
]

MIN_MATCH_SHRINK = 0.05  # reorder.py:32 (applied in csrc/bandk.cpp)


@dataclass(frozen=True, eq=False, repr=False)
class AdjacencyGraph:
    """Undirected graph, CSR adjacency (int64), sorted symmetric rows, no
    self loops; ``edge_weight`` aligned with ``adj_idx``; ``node_weight``
    counts merged rows (reorder.py:35-58)."""

    n_nodes: int
    adj_ptr: np.ndarray
    adj_idx: np.ndarray
    edge_weight: np.ndarray
    node_weight: np.ndarray

    def degrees(self) -> np.ndarray:
        return np.diff(self.adj_ptr)

    def __repr__(self) -> str:
        return f"AdjacencyGraph(n_nodes={self.n_nodes}, n_edges={len(self.adj_idx) // 2})"


@dataclass(frozen=True, eq=False)
class CoarseningMap:
    """Fine node -> coarse node, and each coarse node's fine members in
    ascending order (reorder.py:61-72)."""

    fine_to_coarse: np.ndarray
    coarse_members: list


@dataclass(frozen=True, eq=False)
class BandKResult:
    """Permutation plus per-level group sizes, bottom level first
    (reorder.py:75-84); feeds pack_csrk directly."""

    perm: Permutation
    level_group_sizes: list


def _graph_arrays(g: AdjacencyGraph):
    return (np.ascontiguousarray(g.adj_ptr, dtype=np.int64),
            np.ascontiguousarray(g.adj_idx, dtype=np.int64),
            np.ascontiguousarray(g.edge_weight, dtype=np.int64),
            np.ascontiguousarray(g.node_weight, dtype=np.int64))


def _read_graph(handle) -> tuple:
    sizes = np.zeros(3, dtype=np.int64)
    nat.call("csrk_graph_sizes", handle, nat.i64p(sizes))
    n, m, nf = (int(v) for v in sizes)
    ptr = np.zeros(n + 1, dtype=np.int64)
    idx = np.zeros(m, dtype=np.int64)
    ew = np.zeros(m, dtype=np.int64)
    nw = np.zeros(n, dtype=np.int64)
    f2c = np.zeros(nf, dtype=np.int64)
    nat.call("csrk_graph_get", handle, nat.i64p(ptr), nat.i64p(idx), nat.i64p(ew),
             nat.i64p(nw), nat.i64p(f2c))
    nat.lib().csrk_graph_free(handle)
    return AdjacencyGraph(n, ptr, idx, ew, nw), f2c


def build_graph(a: CsrMatrix) -> AdjacencyGraph:
    """Graph of the pattern of A + A^T without the diagonal, unit weights
    (reorder.py:115-135)."""
    if a.n_rows != a.n_cols:
        raise ValueError("graph construction requires a square matrix")
    out = C.c_void_p()
    nat.call("csrk_build_graph", a.n_rows, nat.u32p(a.row_ptr), nat.u32p(a.col_idx),
             C.byref(out))
    return _read_graph(out)[0]


def heavy_edge_matching(g: AdjacencyGraph) -> np.ndarray:
    """One maximal heavy-edge matching round; partner of each node or the
    node itself (reorder.py:138-173)."""
    ptr, idx, ew, _ = _graph_arrays(g)
    match = np.zeros(g.n_nodes, dtype=np.int64)
    nat.call("csrk_heavy_edge_matching", g.n_nodes, nat.i64p(ptr), nat.i64p(idx),
             nat.i64p(ew), nat.i64p(match))
    return match


def _members(f2c: np.ndarray, m: int) -> list:
    order = np.argsort(f2c, kind="stable")
    cuts = np.searchsorted(f2c[order], np.arange(m + 1))
    return [order[cuts[c]:cuts[c + 1]] for c in range(m)]


def coarsen(g: AdjacencyGraph, target_weight) -> tuple:
    """Repeated heavy-edge matching until the mean coarse weight reaches
    ``target_weight`` or a round shrinks by < 5% (reorder.py:199-237).
    Returns ``(coarse_graph, CoarseningMap)``."""
    if target_weight < 1:
        raise ValueError("target_weight must be at least 1")
    ptr, idx, ew, nw = _graph_arrays(g)
    out = C.c_void_p()
    nat.call("csrk_coarsen", g.n_nodes, nat.i64p(ptr), nat.i64p(idx), nat.i64p(ew),
             nat.i64p(nw), float(target_weight), C.byref(out))
    coarse, f2c = _read_graph(out)
    return coarse, CoarseningMap(f2c, _members(f2c, coarse.n_nodes))


def weighted_bandwidth_order(g: AdjacencyGraph) -> Permutation:
    """Weight-aware reverse Cuthill-McKee order (reorder.py:281-336)."""
    ptr, idx, _, nw = _graph_arrays(g)
    fwd = np.zeros(g.n_nodes, dtype=np.int64)
    nat.call("csrk_weighted_bandwidth_order", g.n_nodes, nat.i64p(ptr), nat.i64p(idx),
             nat.i64p(nw), nat.i64p(fwd))
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(g.n_nodes, dtype=np.int64)
    return Permutation(fwd, inv, _trusted=True)


def _backend(requested):
    """'device' (CUDA, csrc/bandk_dev.cu) or 'host' (C++, csrc/bandk.cpp).
    Both are native and bit-identical; the default is the device when a GPU
    is present (override with CSRK_BANDK_BACKEND)."""
    choice = requested or os.environ.get("CSRK_BANDK_BACKEND", "")
    if choice in ("device", "host"):
        return choice
    if choice:
        raise ValueError(f"unknown band_k backend {choice!r}")
    return "device" if nat.device_count() > 0 else "host"


def band_k(a: CsrMatrix, k: int, level_targets, *, backend: str | None = None) -> BandKResult:
    """Multilevel bandwidth-limiting ordering with super-row (and for k = 3
    super-super-row) derivation (reorder.py:415-469).

    ``level_targets`` = [rows per super-row] or [rows per super-row,
    super-rows per super-super-row].  Realised sizes are powers of two on
    regular grids.  ``backend`` selects the device or host
    native implementation (see :func:`_backend`).
    """
    if k not in (2, 3):
        raise ValueError("k must be 2 or 3")
    targets = [float(t) for t in level_targets]
    if len(targets) != k - 1:
        raise ValueError(f"expected {k - 1} level targets, got {len(targets)}")
    if a.n_rows == 0:
        raise ValueError("cannot reorder an empty matrix")
    if a.n_rows != a.n_cols:
        raise ValueError("graph construction requires a square matrix")
    tarr = np.ascontiguousarray(targets, dtype=np.float64)
    if any(t < 1 for t in targets):
        raise ValueError("target_weight must be at least 1")
    out = C.c_void_p()
    if _backend(backend) == "device":
        nat.call("csrk_band_k_device", a.device().ptr, k, nat.f64p(tarr), C.byref(out))
    else:
        nat.call("csrk_band_k", a.n_rows, nat.u32p(a.row_ptr), nat.u32p(a.col_idx), k,
                 nat.f64p(tarr), C.byref(out))
    try:
        sizes = np.zeros(3, dtype=np.int64)
        nat.call("csrk_bandk_result_sizes", out, nat.i64p(sizes))
        fwd = np.zeros(int(sizes[0]), dtype=np.int64)
        s1 = np.zeros(int(sizes[1]), dtype=np.int64)
        s2 = np.zeros(max(1, int(sizes[2])), dtype=np.int64)
        nat.call("csrk_bandk_result_get", out, nat.i64p(fwd), nat.i64p(s1), nat.i64p(s2))
    finally:
        nat.lib().csrk_bandk_result_free(out)
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(fwd.shape[0], dtype=np.int64)
    levels = [s1.tolist()] if k == 2 else [s1.tolist(), s2[: int(sizes[2])].tolist()]
    return BandKResult(Permutation(fwd, inv, _trusted=True), levels)
