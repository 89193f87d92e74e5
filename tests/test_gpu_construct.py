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


def _hub_graphs():
    """Parents of degree > 128 take the block placement path of the device
    Cuthill-McKee levels: a star, a random graph with hubs, and several
    components of stars and paths."""
    import paper_2203_05096_b200 as ck
    rng = np.random.default_rng(17)
    out = []
    n = 3000  # star: every leaf is a child of the centre
    rows = np.r_[np.zeros(n - 1, dtype=np.int64), np.arange(1, n)]
    cols = np.r_[np.arange(1, n), np.zeros(n - 1, dtype=np.int64)]
    out.append(ck.csr_from_arrays(n, n, rows, cols, np.ones(len(rows))))
    n = 20000  # sparse random graph plus 8 hubs of degree ~1500
    r = rng.integers(0, n, 60000)
    c = rng.integers(0, n, 60000)
    hubs = rng.choice(n, 8, replace=False)
    hr = np.repeat(hubs, 1500)
    hc = rng.integers(0, n, len(hr))
    rows = np.r_[r, c, hr, hc]
    cols = np.r_[c, r, hc, hr]
    out.append(ck.csr_from_arrays(n, n, rows, cols, np.ones(len(rows))))
    parts, off = [], 0  # components: stars of 200..400 leaves and paths
    for k in range(6):
        m = 200 + 40 * k
        if k % 2 == 0:
            rr = np.r_[np.full(m, off), off + 1 + np.arange(m)]
            cc = np.r_[off + 1 + np.arange(m), np.full(m, off)]
        else:
            rr = np.r_[off + np.arange(m), off + 1 + np.arange(m)]
            cc = np.r_[off + 1 + np.arange(m), off + np.arange(m)]
        parts.append((rr, cc))
        off += m + 1
    rows = np.concatenate([p[0] for p in parts])
    cols = np.concatenate([p[1] for p in parts])
    out.append(ck.csr_from_arrays(off, off, rows, cols, np.ones(len(rows))))
    return out


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
    mats.extend(_hub_graphs())
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


def _dev_graph(a):
    dg = C.c_void_p()
    nat.call("csrk_dgraph_build", a.device().ptr, C.byref(dg))
    return dg


def test_device_matching_and_coarsen_match_native(golden):
    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200 import synthetic
    mats = [golden.csr(name) for name in golden.names]
    n, rp, ci, va = synthetic.stencil_arrays((30, 40, 50), 7)
    mats.append(ck.CsrMatrix(n, n, rp, ci, va))
    for a in mats:
        g = ck.build_graph(a)
        dg = _dev_graph(a)
        try:
            match = np.zeros(g.n_nodes, dtype=np.int64)
            iters = C.c_int(0)
            nat.call("csrk_dgraph_match", dg, nat.i64p(match), C.byref(iters))
            np.testing.assert_array_equal(match, ck.heavy_edge_matching(g))
            for target in (2, 3, 7):
                coarse, cmap = ck.coarsen(g, target)
                f2c = np.zeros(g.n_nodes, dtype=np.int64)
                cg = C.c_void_p()
                nat.call("csrk_dgraph_coarsen", dg, float(target), nat.i64p(f2c),
                         C.byref(cg))
                try:
                    np.testing.assert_array_equal(f2c, cmap.fine_to_coarse)
                    _assert_graph_equal(cg, coarse, f"coarsen {target}")
                finally:
                    nat.call("csrk_dgraph_free", cg)
        finally:
            nat.call("csrk_dgraph_free", dg)


def _device_band_k(a, k, targets):
    out = C.c_void_p()
    t = np.ascontiguousarray(targets, dtype=np.float64)
    nat.call("csrk_band_k_device", a.device().ptr, k, nat.f64p(t), C.byref(out))
    try:
        sizes = np.zeros(3, dtype=np.int64)
        nat.call("csrk_bandk_result_sizes", out, nat.i64p(sizes))
        fwd = np.zeros(int(sizes[0]), dtype=np.int64)
        s1 = np.zeros(int(sizes[1]), dtype=np.int64)
        s2 = np.zeros(max(1, int(sizes[2])), dtype=np.int64)
        nat.call("csrk_bandk_result_get", out, nat.i64p(fwd), nat.i64p(s1), nat.i64p(s2))
    finally:
        nat.lib().csrk_bandk_result_free(out)
    return fwd, s1, s2[: int(sizes[2])]


def test_device_band_k_bit_exact_on_golden(golden):
    from conftest import BANDK_TAGS
    for name in golden.names:
        a = golden.csr(name)
        for tag, k, targets in BANDK_TAGS:
            fwd, s1, s2 = _device_band_k(a, k, targets)
            np.testing.assert_array_equal(fwd, golden[f"{name}/{tag}/fwd"],
                                          err_msg=f"{name} {tag}")
            np.testing.assert_array_equal(s1, golden[f"{name}/{tag}/sizes0"])
            if k == 3:
                np.testing.assert_array_equal(s2, golden[f"{name}/{tag}/sizes1"])


@pytest.mark.parametrize("name", ["grid2d_200", "grid3d7_32", "grid3d27_20", "irregular_200k",
                                  "C1"])
def test_device_band_k_digests(name, configs_golden):
    import paper_2203_05096_b200 as ck
    from conftest import digest
    from paper_2203_05096_b200 import synthetic
    rec = configs_golden[name]
    spec = rec["spec"]
    if spec["kind"] == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays(spec["shape"], spec["points"],
                                                 values=spec.get("values", "laplacian"))
        a = ck.CsrMatrix(n, n, rp, ci, va)
    else:
        r, c, v = synthetic.irregular_triplets(spec["rows"], seed=spec.get("seed", 0))
        a = ck.csr_from_arrays(spec["rows"], spec["rows"], r, c, v)
    for run in rec["runs"]:
        fwd, s1, s2 = _device_band_k(a, 3, run["targets"])
        assert digest(fwd, "<i8") == run["fwd"]
        assert digest(s1, "<i8") == run["sizes0"]
        assert digest(s2, "<i8") == run["sizes1"]


@pytest.mark.parametrize("case", ["dups", "long_runs", "zeros", "wide"])
def test_device_coo_to_csr_bitwise(monkeypatch, case):
    """csrk_coo_to_csr equals the host restatement of csr_from_arrays
    (reference format.py:233-284) bit for bit: stable (row, col) order and
    duplicates summed as np.add.reduceat does (runs of 1..500)."""
    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200 import format as F
    rng = np.random.default_rng(len(case))
    if case == "dups":
        n_rows, n_cols, count = 70001, 3001, 400000
        r = rng.integers(0, n_rows, count)
        c = rng.integers(0, n_cols, count)
        v = rng.standard_normal(count) * 10.0 ** rng.uniform(-8, 8, count)
    elif case == "long_runs":  # the same coordinate 1..500 times
        n_rows, n_cols = 1000, 1000
        lens = rng.integers(1, 500, 600)
        r = np.repeat(rng.integers(0, n_rows, 600), lens)
        c = np.repeat(rng.integers(0, n_cols, 600), lens)
        v = rng.standard_normal(len(r)) * 10.0 ** rng.uniform(-12, 12, len(r))
        perm = rng.permutation(len(r))
        r, c, v = r[perm], c[perm], v[perm]
    elif case == "zeros":  # signed zeros and cancellation
        n_rows, n_cols, count = 50000, 50000, 200000
        r = rng.integers(0, 300, count)
        c = rng.integers(0, 300, count)
        v = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, 1e-300, -3.0]), count)
    else:  # wide: 32-bit columns, most rows empty
        n_rows, n_cols, count = 3_000_000, 4_000_000_000, 300000
        r = rng.integers(0, n_rows, count)
        c = rng.integers(0, n_cols, count)
        v = rng.uniform(-1, 1, count)
    monkeypatch.setattr(F, "DEVICE_COO_MIN", 1 << 62)
    want = ck.csr_from_arrays(n_rows, n_cols, r, c, v)
    monkeypatch.setattr(F, "DEVICE_COO_MIN", 1)
    got = ck.csr_from_arrays(n_rows, n_cols, r, c, v)
    assert got._dev is not None
    np.testing.assert_array_equal(got.row_ptr, want.row_ptr)
    np.testing.assert_array_equal(got.col_idx, want.col_idx)
    assert np.array_equal(got.vals.view(np.uint64), want.vals.view(np.uint64))
    # the attached device copy is the same matrix
    rp, ci, va, _, _ = got.device().download()
    np.testing.assert_array_equal(rp, want.row_ptr)
    np.testing.assert_array_equal(va, want.vals)
