"""Host-side behaviour of the drop-in API (no GPU needed): containers and
their validation messages, native Band-k against the reference's outputs,
the tuning model tables, profiles, search and timing protocol.  Mirrors the
reference's own tests (pkg/tests/test_format.py, test_reorder.py,
test_tuning.py, test_bench.py)."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from conftest import BANDK_TAGS, random_csr, tridiagonal

# ---- format --------------------------------------------------------------


def test_build_csr_canonical_and_duplicates():
    a = ck.build_csr(2, 2, [(0, 0, 1.0), (0, 0, 2.0)])
    assert a.nnz == 1 and a.vals.tolist() == [3.0] and a.row_ptr.tolist() == [0, 1, 1]
    z = ck.build_csr(2, 2, [(0, 1, 0.0)])
    assert z.nnz == 1 and z.vals.tolist() == [0.0]
    e = ck.build_csr(3, 3, [])
    assert e.row_ptr.tolist() == [0, 0, 0, 0]
    assert ck.build_csr(0, 0, []).row_ptr.tolist() == [0]
    assert a.row_ptr.dtype == np.uint32 and a.col_idx.dtype == np.uint32
    assert a.vals.dtype == np.float64


def test_csr_from_arrays_matches_reference_on_golden_inputs(golden):
    # the golden CSR arrays were produced by the reference csr_from_arrays;
    # rebuilding from their COO triplets in scrambled order must reproduce them
    rng = np.random.default_rng(3)
    for name in golden.names[:30]:
        a = golden.csr(name)
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.astype(np.int64)))
        order = rng.permutation(a.nnz)
        b = ck.csr_from_arrays(a.n_rows, a.n_cols, rows[order],
                               a.col_idx[order].astype(np.int64), a.vals[order])
        np.testing.assert_array_equal(b.row_ptr, a.row_ptr)
        np.testing.assert_array_equal(b.col_idx, a.col_idx)
        np.testing.assert_array_equal(b.vals, a.vals)


def test_csr_from_arrays_errors_name_position():
    with pytest.raises(ValueError, match="triplet 1"):
        ck.build_csr(2, 2, [(0, 0, 1.0), (5, 0, 1.0)])
    with pytest.raises(ValueError, match="column index"):
        ck.build_csr(2, 2, [(0, 3, 1.0)])
    with pytest.raises(ValueError, match="equal length"):
        ck.csr_from_arrays(2, 2, [0], [0, 1], [1.0])


def test_csr_validation_messages():
    ok = dict(n_rows=2, n_cols=2, row_ptr=np.array([0, 1, 2]), col_idx=np.array([0, 1]),
              vals=np.array([1.0, 2.0]))
    ck.CsrMatrix(**ok)
    for bad, msg in ((dict(ok, row_ptr=np.array([1, 1, 2])), "row_ptr\\[0\\]"),
                     (dict(ok, row_ptr=np.array([0, 2, 1])), "non-decreasing"),
                     (dict(ok, col_idx=np.array([0, 5])), "out of range"),
                     (dict(ok, row_ptr=np.array([0, 2, 2]), col_idx=np.array([1, 0])),
                      "increasing"),
                     (dict(ok, row_ptr=np.array([0, 2, 2]), col_idx=np.array([1, 1])),
                      "increasing"),
                     (dict(ok, n_rows=-1), "non-negative")):
        with pytest.raises(ValueError, match=msg):
            ck.CsrMatrix(**bad)


def test_storage_is_immutable():
    a = ck.build_csr(2, 2, [(0, 0, 1.0)])
    with pytest.raises(ValueError):
        a.vals[0] = 7.0
    with pytest.raises(AttributeError):
        a.n_rows = 3


def test_permutation_validation_and_constructors():
    ck.Permutation(fwd=np.array([1, 0]), inv=np.array([1, 0]))
    with pytest.raises(ValueError):
        ck.Permutation(fwd=np.array([1, 0]), inv=np.array([0, 1]))
    with pytest.raises(ValueError):
        ck.Permutation(fwd=np.array([0, 0]), inv=np.array([0, 0]))
    q = ck.Permutation.from_forward([2, 0, 1])
    assert q.inv.tolist() == [1, 2, 0] and len(q) == 3
    assert ck.Permutation.identity(4).fwd.tolist() == [0, 1, 2, 3]


def test_csrk_matrix_validation():
    a = tridiagonal(9, 42)
    with pytest.raises(ValueError):
        ck.CsrKMatrix(a, 2, (np.array([0, 4, 3, 9]),), ck.Permutation.identity(9))
    with pytest.raises(ValueError, match="level 1"):
        ck.CsrKMatrix(a, 2, (np.array([0, 4, 8]),), ck.Permutation.identity(9))
    with pytest.raises(ValueError, match="k must be 2 or 3"):
        ck.CsrKMatrix(a, 4, (), ck.Permutation.identity(9))
    m = ck.CsrKMatrix(a, 3, (np.array([0, 2, 5, 7, 9]), np.array([0, 2, 4])),
                      ck.Permutation.identity(9))
    assert m.sr_ptr.tolist() == [0, 2, 5, 7, 9] and m.ssr_ptr.tolist() == [0, 2, 4]
    assert m.sr_ptr.dtype == np.uint32 and m.num_super_rows == 4 and m.num_ssr == 2
    assert m.as_csr() is a
    m2 = ck.CsrKMatrix(a, 2, (np.array([0, 9]),), ck.Permutation.identity(9))
    with pytest.raises(AttributeError):
        _ = m2.ssr_ptr


def test_pack_rejects_bad_groupings_before_device_work():
    a = tridiagonal(9, 42)
    p = ck.Permutation.identity(9)
    with pytest.raises(ValueError, match="level 1"):
        ck.pack_csrk(a, p, [[2, 3, 2]])
    with pytest.raises(ValueError, match="level 2"):
        ck.pack_csrk(a, p, [[2, 3, 2, 2], [2, 3]])
    with pytest.raises(ValueError):
        ck.pack_csrk(a, p, [])
    with pytest.raises(ValueError):
        ck.pack_csrk(a, p, [[9], [1], [1]])
    with pytest.raises(ValueError):
        ck.pack_csrk(a, p, [[0, 9]])
    with pytest.raises(ValueError, match="square"):
        ck.pack_csrk(ck.build_csr(2, 3, [(0, 0, 1.0)]), ck.Permutation.identity(2), [[2]])


def test_vector_length_checks():
    p = ck.Permutation.identity(3)
    with pytest.raises(ValueError):
        ck.permute_vector(p, np.zeros(4))
    with pytest.raises(ValueError):
        ck.unpermute_vector(p, np.zeros(2))


# ---- native Band-k -------------------------------------------------------


def test_band_k_bit_exact_on_golden_cases(golden):
    for name in golden.names:
        a = golden.csr(name)
        for tag, k, targets in BANDK_TAGS:
            res = ck.band_k(a, k, targets)
            np.testing.assert_array_equal(res.perm.fwd, golden[f"{name}/{tag}/fwd"],
                                          err_msg=f"{name} {tag}")
            for lv, sizes in enumerate(res.level_group_sizes):
                assert sizes == golden[f"{name}/{tag}/sizes{lv}"].tolist()


def test_graph_functions_bit_exact_on_golden_cases(golden):
    for name in golden.names:
        a = golden.csr(name)
        g = ck.build_graph(a)
        np.testing.assert_array_equal(g.adj_ptr, golden[f"{name}/graph_ptr"])
        np.testing.assert_array_equal(g.adj_idx, golden[f"{name}/graph_idx"])
        np.testing.assert_array_equal(ck.heavy_edge_matching(g), golden[f"{name}/hem"])
        np.testing.assert_array_equal(ck.weighted_bandwidth_order(g).fwd,
                                      golden[f"{name}/wbo_fwd"])
        for t in (2, 3):
            cg, cmap = ck.coarsen(g, t)
            np.testing.assert_array_equal(cmap.fine_to_coarse, golden[f"{name}/coarsen{t}_f2c"])
            np.testing.assert_array_equal(cg.adj_ptr, golden[f"{name}/coarsen{t}_ptr"])
            np.testing.assert_array_equal(cg.adj_idx, golden[f"{name}/coarsen{t}_idx"])
            np.testing.assert_array_equal(cg.edge_weight, golden[f"{name}/coarsen{t}_ew"])
            np.testing.assert_array_equal(cg.node_weight, golden[f"{name}/coarsen{t}_nw"])
            for c, members in enumerate(cmap.coarse_members):
                assert np.all(cmap.fine_to_coarse[members] == c)


def test_band_k_reference_properties():
    # pkg/tests/test_reorder.py:160-169: tridiagonal(8), target 2
    a = tridiagonal(8)
    res = ck.band_k(a, 2, [2])
    assert res.level_group_sizes[0] == [2, 2, 2, 2]
    rows = np.repeat(np.arange(8), np.diff(a.row_ptr.astype(np.int64)))
    fwd = res.perm.fwd
    assert int(np.abs(fwd[rows] - fwd[a.col_idx.astype(np.int64)]).max()) == 1
    # coarsening a path gives pairs (test_reorder.py:87-93)
    path = ck.build_graph(ck.build_csr(4, 4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)]))
    coarse, cmap = ck.coarsen(path, 2)
    assert coarse.node_weight.tolist() == [2, 2]
    assert [sorted(m.tolist()) for m in cmap.coarse_members] == [[0, 1], [2, 3]]


def test_band_k_argument_errors():
    a = tridiagonal(9, 42)
    with pytest.raises(ValueError):
        ck.band_k(a, 4, [2, 2, 2])
    with pytest.raises(ValueError):
        ck.band_k(a, 3, [2])
    with pytest.raises(ValueError):
        ck.band_k(ck.build_csr(0, 0, []), 2, [2])
    with pytest.raises(ValueError):
        ck.coarsen(ck.build_graph(a), 0)
    with pytest.raises(ValueError):
        ck.build_graph(ck.build_csr(2, 3, [(0, 0, 1.0)]))


def test_band_k_random_inputs_are_valid_permutations():
    rng = np.random.default_rng(8)
    for _ in range(40):
        n = int(rng.integers(1, 60))
        a = random_csr(rng, n, n, float(rng.uniform(0.02, 0.3)))
        for k, targets in ((2, [2]), (3, [2, 2])):
            res = ck.band_k(a, k, targets)
            assert sorted(res.perm.fwd.tolist()) == list(range(n))
            assert sum(res.level_group_sizes[0]) == n
            if k == 3:
                assert sum(res.level_group_sizes[1]) == len(res.level_group_sizes[0])


# ---- tuning model --------------------------------------------------------

VOLTA_TABLE = {1: (9, 10), 8: (6, 7), 16: (8, 12), 20: (20, 10), 32: (20, 10), 100: (15, 7)}
AMPERE_TABLE = {1: (9, 21), 8: (6, 13), 16: (6, 44), 20: (13, 39), 32: (13, 39), 100: (6, 12)}


def _stats(rd, var=0.0):
    return ck.MatrixStats(n=100, nnz=int(rd * 100), rdensity=rd, variance=var,
                          max_row_nnz=int(rd) + 1, pattern_symmetry=1.0)


def test_size_tables_match_reference():
    for profile, table in ((ck.VOLTA, VOLTA_TABLE), (ck.AMPERE, AMPERE_TABLE)):
        for rd, want in table.items():
            case, _ = ck.select_case(float(rd))
            assert ck.adjust_sizes(profile, case, *ck.base_sizes(profile, float(rd))) == want
            p = ck.tune_gpu(_stats(float(rd)), profile)
            assert (p.ssrs, p.srs) == want


def test_case_boundaries_and_dims():
    assert [ck.select_case(v)[0] for v in (6.93, 8.0, 8.000001, 16.0, 16.5, 32.0, 34.65)] == \
        [1, 1, 2, 2, 3, 3, 4]
    assert ck.select_case(10.0)[1] == ck.BlockDims(4, 8, 12)
    with pytest.raises(ValueError):
        ck.select_case(0.0)


def test_round_half_up_and_classification():
    assert [ck.round_half_up(v) for v in (2.4, 2.5, 7.5, -0.5, -1.5)] == [2, 3, 8, 0, -1]
    assert ck.classify(_stats(4.0, 10.0)) is ck.MatrixClass.REGULAR
    assert ck.classify(_stats(4.0, float(np.nextafter(10.0, 11.0)))) is ck.MatrixClass.IRREGULAR


def test_tune_variants_and_params():
    assert ck.tune_gpu(_stats(2.15), ck.VOLTA).kernel_variant is ck.KernelVariant.GPU3
    assert ck.tune_gpu(_stats(8.0), ck.VOLTA).kernel_variant is ck.KernelVariant.GPU3
    p = ck.tune_gpu(_stats(14.34), ck.VOLTA)
    assert p.kernel_variant is ck.KernelVariant.GPU35 and p.block_dims == ck.BlockDims(4, 8, 12)
    assert ck.tune_gpu(_stats(1.0), ck.VOLTA).to_dict() == {
        "k": 3, "ssrs": 9, "srs": 10, "block_dims": [8, 12, 1], "kernel_variant": "gpu3-emu"}
    assert ck.tune_cpu(_stats(50.0, 400.0)).to_dict() == {
        "k": 2, "ssrs": None, "srs": 96, "block_dims": None, "kernel_variant": "cpu2"}
    b = ck.tune_gpu(_stats(6.98), ck.b200_profile())
    assert b.kernel_variant is ck.KernelVariant.CUDA3
    with pytest.raises(ValueError, match="block"):
        ck.TuningParams(k=3, ssrs=7, srs=8, block_dims=None,
                        kernel_variant=ck.KernelVariant.CUDA3)


def test_candidate_sets():
    ladder = (4, 6, 8, 12, 16, 24, 32, 48)
    grid = ck.gpu_candidate_grid()
    assert len(grid) == 64 and set(grid) == {(a, b) for a in ladder for b in ladder}
    srs = ck.cpu_candidate_srs()
    assert len(srs) == 18 and srs[0] == 8 and srs[-1] == 3072 and 96 in srs
    assert ck.cpu_fallback_srs() == 96
    assert all(s & (s - 1) == 0 for pair in ck.b200_candidate_grid() for s in pair)


def test_grid_search_and_fit():
    a = ck.build_csr(1, 1, [(0, 0, 1.0)])
    r = ck.grid_search(a, [3, 1, 2], lambda m, c: 1.0, reps=2)
    assert r.best == 1 and [c for c, _ in r.table] == [1, 2, 3]
    calls = []
    ck.grid_search(a, [1, 2, 3], lambda m, c: calls.append(c) or 1.0, reps=4)
    assert len(calls) == 12
    assert ck.grid_search(a, ck.cpu_candidate_srs(),
                          lambda m, c: abs(c - 100) * 1e-6 + 1e-9, reps=3).best == 96
    with pytest.raises(ValueError):
        ck.grid_search(a, [], lambda m, c: 1.0)
    samples = [(rd, 8.9 - 1.25 * math.log(rd)) for rd in (1.0, 2.0, 4.0, 10.0, 33.0)]
    fa, fb = ck.fit_log_model(samples)
    assert abs(fa - 8.9) <= 1e-9 and abs(fb - 1.25) <= 1e-9
    assert ck.fit_log_model([(1.0, 9.0), (math.e, 8.0)], b_override=1.25)[1] == 1.25
    with pytest.raises(ValueError):
        ck.fit_log_model([(2.0, 5.0), (2.0, 6.0)])


def test_profiles_round_trip(tmp_path):
    import os

    from paper_2203_05096_b200 import tuning
    data = os.path.join(os.path.dirname(tuning.__file__), "data")
    assert ck.load_profile(os.path.join(data, "volta.json")) == ck.VOLTA
    assert ck.load_profile(os.path.join(data, "ampere.json")) == ck.AMPERE
    for prof in (ck.VOLTA, ck.AMPERE, ck.b200_profile()):
        assert ck.profile_from_dict(ck.profile_to_dict(prof)) == prof
        path = tmp_path / f"{prof.name}.json"
        ck.save_profile(prof, path)
        assert ck.load_profile(path) == prof
    with pytest.raises(ValueError):
        ck.DeviceProfile("bad", (1, 1), (1, 1), (
            ck.CaseRule(16.0, ck.BlockDims(8, 12)), ck.CaseRule(8.0, ck.BlockDims(8, 12)),
            ck.CaseRule(None, ck.BlockDims(8, 12))))


# ---- kernels / bench host logic -------------------------------------------


def test_block_dims_and_trace():
    with pytest.raises(ValueError):
        ck.BlockDims(0, 1)
    with pytest.raises(ValueError, match="1024"):
        ck.BlockDims(32, 32, 2)
    t = ck.EmulationTrace.from_records([(0, 0, 0, 0, 0, 1, 0), (0, 0, 0, 1, 0, 1, 0)])
    with pytest.raises(ValueError):
        t.validate_partition(2)
    ck.EmulationTrace.from_records([(1, 0, 0, 0, 0, 1, 0), (0, 0, 0, 1, 0, 1, 0)]) \
        .validate_partition(2)


def test_kernel_argument_checks_precede_device_work():
    a = tridiagonal(9, 42)
    m = ck.CsrKMatrix(a, 3, (np.array([0, 2, 5, 7, 9]), np.array([0, 2, 4])),
                      ck.Permutation.identity(9))
    m2 = ck.CsrKMatrix(a, 2, (np.array([0, 9]),), ck.Permutation.identity(9))
    with pytest.raises(ValueError, match="k"):
        ck.spmv_csr2(m, np.ones(9))
    with pytest.raises(ValueError, match="k"):
        ck.spmv_csr3(m2, np.ones(9))
    with pytest.raises(ValueError, match="z"):
        ck.emulate_gpu_spmv3(m, np.ones(9), ck.BlockDims(8, 12, 2))
    with pytest.raises(ValueError, match="k"):
        ck.emulate_gpu_spmv35(m2, np.ones(9), ck.BlockDims(1, 1, 1))
    with pytest.raises(ValueError, match="length"):
        ck.spmv_csr_ref(a, np.ones(5))


def test_time_kernel_protocol():
    import itertools
    counter = itertools.count()
    calls = []
    durations, last = ck.time_kernel(lambda: calls.append(0) or len(calls), warmups=5,
                                     reps=20, clock=lambda: float(next(counter)))
    assert len(calls) == 25 and durations == [1.0] * 20 and last == 25
    with pytest.raises(ValueError):
        ck.time_kernel(lambda: None, warmups=-1, reps=5)
    with pytest.raises(ValueError):
        ck.time_kernel(lambda: None, warmups=5, reps=0)
    assert (ck.DEFAULT_WARMUPS, ck.DEFAULT_REPS, ck.DEFAULT_TOLERANCE) == (5, 20, 1e-10)


def test_error_metrics_and_targets():
    from paper_2203_05096_b200.bench import TARGETS, scaled_error, spmv_bytes
    assert ck.max_rel_error(np.zeros(3), np.zeros(3)) == 0.0
    assert ck.max_rel_error(np.array([1.1]), np.array([1.0])) == pytest.approx(0.1)
    with pytest.raises(ValueError):
        ck.max_rel_error(np.zeros(2), np.zeros(3))
    assert TARGETS[:5] == ("ref", "cpu2", "cpu3", "gpu3-emu", "gpu35-emu")
    assert {"cuda3", "cuda35"} <= set(TARGETS)
    assert scaled_error([1.0, 2.0], [1.0, 2.0 + 1e-12], [1.0, 4.0]) == pytest.approx(2.5e-13)
    # C2 fp64 moves 1,740.1 MB per SpMV
    assert spmv_bytes(16_777_216, 16_777_216, 117_047_296) == pytest.approx(1_740.1e6, rel=1e-4)
    with pytest.raises(ValueError):
        ck.run_benchmark(tridiagonal(4), "x", "cuda9000", warmups=0, reps=1)


def test_default_threads_env(monkeypatch):
    monkeypatch.setenv("OMP_NUM_THREADS", "7")
    assert ck.default_threads() == 7
    monkeypatch.setenv("OMP_NUM_THREADS", "0")
    assert ck.default_threads() >= 1
