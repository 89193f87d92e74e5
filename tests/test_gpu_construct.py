"""Device construction primitives: the stable radix sort used by device-side
graph building (checked against numpy's stable argsort)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2203_05096_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _device_sort(keys, vals, begin, end):
    kd = nat.DeviceBuffer.from_array(keys)
    vd = nat.DeviceBuffer.from_array(vals)
    nat.call("csrk_sort_pairs", nat.current_device(), len(keys), kd.ptr, vd.ptr, begin, end,
             None)
    nat.call("csrk_stream_sync", None)
    return kd.to_array(np.uint64, len(keys)), vd.to_array(np.uint32, len(keys))


@pytest.mark.parametrize("n,bits,spread", [(1, 64, 10), (1000, 64, 50), (5000, 16, 30),
                                           (300_000, 64, 2 ** 40), (70_000, 32, 7)])
def test_radix_sort_is_stable_and_exact(n, bits, spread):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, spread, n, dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint32)
    sk, sv = _device_sort(keys, vals, 0, bits)
    mask = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    order = np.argsort(keys & mask, kind="stable")
    np.testing.assert_array_equal(sv, vals[order])
    np.testing.assert_array_equal(sk, keys[order])


def _dgraph_arrays(handle):
    sz = np.zeros(2, dtype=np.int64)
    nat.call("csrk_dgraph_sizes", handle, nat.i64p(sz))
    n, m = int(sz[0]), int(sz[1])
    ptr = np.zeros(n + 1, dtype=np.int64)
    idx = np.zeros(m, dtype=np.int64)
    ew = np.zeros(m, dtype=np.int64)
    nw = np.zeros(n, dtype=np.int64)
    nat.call("csrk_dgraph_download", handle, nat.i64p(ptr), nat.i64p(idx), nat.i64p(ew),
             nat.i64p(nw))
    return ptr, idx, ew, nw


def _assert_graph_equal(handle, g, msg=""):
    ptr, idx, ew, nw = _dgraph_arrays(handle)
    np.testing.assert_array_equal(ptr, g.adj_ptr, err_msg=msg)
    np.testing.assert_array_equal(idx, g.adj_idx, err_msg=msg)
    np.testing.assert_array_equal(ew, g.edge_weight, err_msg=msg)
    np.testing.assert_array_equal(nw, g.node_weight, err_msg=msg)


def test_device_graph_build_relabel_contract(golden):
    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200 import synthetic
    cases = [golden.csr(name) for name in golden.names[:40]]
    n, rp, ci, va = synthetic.stencil_arrays((60, 70, 80), 7)
    cases.append(ck.CsrMatrix(n, n, rp, ci, va))
    for a in cases:
        g = ck.build_graph(a)
        dg = C.c_void_p()
        nat.call("csrk_dgraph_build", a.device().ptr, C.byref(dg))
        try:
            _assert_graph_equal(dg, g, "build")
            perm = ck.weighted_bandwidth_order(g)
            rl = C.c_void_p()
            fwd = np.ascontiguousarray(perm.fwd)
            nat.call("csrk_dgraph_relabel", dg, nat.i64p(fwd), C.byref(rl))
            # host relabel through coarsen(target 1) is the identity; compare with
            # the explicit definition instead: row i of the result is row inv[i]
            ptr, idx, ew, nw = _dgraph_arrays(rl)
            inv = perm.inv
            for i in range(0, g.n_nodes, max(1, g.n_nodes // 97)):
                v = inv[i]
                row = sorted(zip(fwd[g.adj_idx[g.adj_ptr[v]:g.adj_ptr[v + 1]]].tolist(),
                                 g.edge_weight[g.adj_ptr[v]:g.adj_ptr[v + 1]].tolist()))
                got = list(zip(idx[ptr[i]:ptr[i + 1]].tolist(), ew[ptr[i]:ptr[i + 1]].tolist()))
                assert got == row
            np.testing.assert_array_equal(nw, g.node_weight[inv])
            nat.call("csrk_dgraph_free", rl)
            # contraction by coarsen's final fine-to-coarse map reproduces the
            # coarse graph (contraction composes; weights are sums)
            for target in (2, 4):
                coarse, cmap = ck.coarsen(g, target)
                f2c = np.ascontiguousarray(cmap.fine_to_coarse)
                ct = C.c_void_p()
                nat.call("csrk_dgraph_contract", dg, nat.i64p(f2c), coarse.n_nodes,
                         C.byref(ct))
                try:
                    _assert_graph_equal(ct, coarse, f"contract {target}")
                finally:
                    nat.call("csrk_dgraph_free", ct)
        finally:
            nat.call("csrk_dgraph_free", dg)


def test_device_wbo_matches_native(golden):
    """Level-synchronous device RCM equals the sequential order exactly, on
    the golden graphs (many have several components / isolated nodes), on a
    3-D grid and on weighted coarse graphs."""
    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200 import synthetic
    mats = [golden.csr(name) for name in golden.names]
    n, rp, ci, va = synthetic.stencil_arrays((40, 45, 50), 7)
    mats.append(ck.CsrMatrix(n, n, rp, ci, va))
    n, rp, ci, va = synthetic.stencil_arrays((300, 300), 5)
    mats.append(ck.CsrMatrix(n, n, rp, ci, va))
    for a in mats:
        g = ck.build_graph(a)
        dg = C.c_void_p()
        nat.call("csrk_dgraph_build", a.device().ptr, C.byref(dg))
        try:
            fwd = np.zeros(g.n_nodes, dtype=np.int64)
            nat.call("csrk_dgraph_wbo", dg, nat.i64p(fwd))
            np.testing.assert_array_equal(fwd, ck.weighted_bandwidth_order(g).fwd)
            if g.n_nodes >= 4:
                coarse, cmap = ck.coarsen(g, 3)
                ct = C.c_void_p()
                f2c = np.ascontiguousarray(cmap.fine_to_coarse)
                nat.call("csrk_dgraph_contract", dg, nat.i64p(f2c), coarse.n_nodes,
                         C.byref(ct))
                try:
                    cf = np.zeros(coarse.n_nodes, dtype=np.int64)
                    nat.call("csrk_dgraph_wbo", ct, nat.i64p(cf))
                    np.testing.assert_array_equal(cf, ck.weighted_bandwidth_order(coarse).fwd)
                finally:
                    nat.call("csrk_dgraph_free", ct)
        finally:
            nat.call("csrk_dgraph_free", dg)
