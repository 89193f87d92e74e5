"""Generate the golden fixtures that pin this repo to the reference ``csrk``.

Run in the build container, where the read-only reference lives at
/root/reference (it does not exist on the GPU box, so its outputs travel as
the committed files this script writes):

    python tests/golden/make_golden.py small      # ~1 min  -> small_cases.npz
    python tests/golden/make_golden.py medium     # ~2 min  -> configs.json
    python tests/golden/make_golden.py large      # ~20 min -> configs.json
    python tests/golden/make_golden.py b200 [C2 C3 C5 C1]   # adds runs at the
                                                  # B200 profile's targets
    python tests/golden/make_golden.py mm         # ~20 s  -> mm.json (Matrix
                                                  # Market ingest, mm_cases.py)

``small`` stores full arrays for many small matrices (the shapes of the
reference's own sweep, pkg/tests/test_acceptance.py:86-154, plus the kernel
fixtures of pkg/tests/test_kernels.py).  ``medium``/``large`` store SHA-256
digests of every integer array and every y for the BASELINE configs, so the
full-size device results can be checked bit for bit without shipping GBs.

Every output is produced by the UNMODIFIED reference package imported from
/root/reference/pkg/src; only the input generators come from this repo.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import csrk as ref  # noqa: E402  (the reference package)

_spec = importlib.util.spec_from_file_location(
    "_synthetic", os.path.join(REPO, "paper_2203_05096_b200", "synthetic.py"))
synthetic = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synthetic)


def digest(arr, dtype) -> str:
    a = np.ascontiguousarray(np.asarray(arr).astype(dtype, copy=False))
    return hashlib.sha256(a.tobytes()).hexdigest()


# ----------------------------------------------------------------------------
# small: full arrays
# ----------------------------------------------------------------------------

def _coo(a):
    counts = np.diff(a.row_ptr.astype(np.int64))
    return (np.repeat(np.arange(a.n_rows, dtype=np.int64), counts),
            a.col_idx.astype(np.int64))


def _random_csr(rng, n_rows, n_cols, density, lo=0.5, hi=1.5):
    want = min(max(0, int(round(density * n_rows * n_cols))), n_rows * n_cols)
    flat = rng.choice(n_rows * n_cols, size=want, replace=False)
    return ref.csr_from_arrays(n_rows, n_cols, (flat // n_cols).astype(np.int64),
                               (flat % n_cols).astype(np.int64),
                               rng.uniform(lo, hi, size=want))


def _sweep_case(seed):
    """Four structural shapes: random, block-diagonal, empty rows, dense row."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 121))
    density = float(rng.uniform(0.01, 0.08))
    kind = seed % 4
    if kind == 0:
        return _random_csr(rng, n, n, density)
    if kind == 1:
        n1 = int(rng.integers(1, n))
        b1 = _random_csr(rng, n1, n1, density)
        b2 = _random_csr(rng, n - n1, n - n1, density)
        r1, c1 = _coo(b1)
        r2, c2 = _coo(b2)
        rows = np.concatenate([r1, r2 + n1])
        cols = np.concatenate([c1, c2 + n1])
        return ref.csr_from_arrays(n, n, rows, cols, rng.uniform(0.5, 1.5, len(rows)))
    if kind == 2:
        a0 = _random_csr(rng, n, n, density)
        rows, cols = _coo(a0)
        holes = rng.choice(n, size=max(1, n // 10), replace=False)
        keep = ~np.isin(rows, holes)
        return ref.csr_from_arrays(n, n, rows[keep], cols[keep],
                                   rng.uniform(0.5, 1.5, int(keep.sum())))
    a0 = _random_csr(rng, n, n, density)
    rows, cols = _coo(a0)
    dense_row = int(rng.integers(0, n))
    keep = rows != dense_row
    rows = np.concatenate([rows[keep], np.full(n, dense_row, dtype=np.int64)])
    cols = np.concatenate([cols[keep], np.arange(n, dtype=np.int64)])
    return ref.csr_from_arrays(n, n, rows, cols, rng.uniform(-1.0, 1.0, len(rows)))


EMU35_DIMS = [(4, 8, 12), (8, 8, 8), (16, 8, 4), (2, 2, 2), (3, 5, 2), (1, 3, 4), (32, 2, 2)]
EMU3_DIMS = [(8, 12, 1), (1, 1, 1), (5, 3, 1)]
# y of these emu35 dims is stored for both x vectors; the rest only for x_sgn
EMU35_BOTH = {(4, 8, 12), (3, 5, 2)}


def _store_csr(out, key, a):
    out[f"{key}/shape"] = np.array([a.n_rows, a.n_cols], dtype=np.int64)
    out[f"{key}/row_ptr"] = a.row_ptr
    out[f"{key}/col_idx"] = a.col_idx
    out[f"{key}/vals"] = a.vals


def small():
    out = {}
    cases = []
    # kernel fixtures (pkg/tests/test_kernels.py:31-46, conftest.py:59-69)
    small4 = ref.build_csr(4, 4, [(0, 0, 2.0), (0, 2, 1.0), (1, 1, 3.0), (2, 2, 4.0),
                                  (2, 3, 5.0), (3, 0, 1.0), (3, 3, 6.0)])
    fig1 = synthetic_tridiagonal(9, 42)
    cases.append(("small4", small4))
    cases.append(("fig1", fig1))
    for s in range(64):
        cases.append((f"sweep{s}", _sweep_case(s)))
    # a row longer than one warp and a graph with isolated nodes
    rng = np.random.default_rng(77)
    cases.append(("dense40", _random_csr(rng, 40, 40, 0.9, -1.0, 1.0)))
    cases.append(("diag7", ref.build_csr(7, 7, [(i, i, float(i + 1)) for i in range(7)])))
    names = []
    for name, a in cases:
        names.append(name)
        _store_csr(out, name, a)
        n = a.n_rows
        rng = np.random.default_rng(len(names))
        xp_pos = rng.uniform(0.5, 1.5, n)
        xp_sgn = rng.uniform(-1.0, 1.0, n)
        out[f"{name}/x_pos"] = xp_pos
        out[f"{name}/x_sgn"] = xp_sgn
        out[f"{name}/y_ref_pos"] = ref.spmv_csr_ref(a, xp_pos)
        out[f"{name}/y_ref_sgn"] = ref.spmv_csr_ref(a, xp_sgn)
        st = ref.compute_stats(a)
        out[f"{name}/stats"] = np.array([st.rdensity, st.variance, st.pattern_symmetry,
                                         st.max_row_nnz], dtype=np.float64)
        g = ref.build_graph(a)
        out[f"{name}/graph_ptr"] = g.adj_ptr
        out[f"{name}/graph_idx"] = g.adj_idx
        out[f"{name}/hem"] = ref.heavy_edge_matching(g)
        out[f"{name}/wbo_fwd"] = ref.weighted_bandwidth_order(g).fwd
        for t in (2, 3):
            cg, cmap = ref.coarsen(g, t)
            out[f"{name}/coarsen{t}_f2c"] = cmap.fine_to_coarse
            out[f"{name}/coarsen{t}_ptr"] = cg.adj_ptr
            out[f"{name}/coarsen{t}_idx"] = cg.adj_idx
            out[f"{name}/coarsen{t}_ew"] = cg.edge_weight
            out[f"{name}/coarsen{t}_nw"] = cg.node_weight
        for k, targets in ((2, [4]), (3, [4, 2]), (3, [2, 3]), (3, [8, 4])):
            tag = f"k{k}_" + "_".join(str(t) for t in targets)
            res = ref.band_k(a, k, targets)
            out[f"{name}/{tag}/fwd"] = res.perm.fwd
            for lv, sizes in enumerate(res.level_group_sizes):
                out[f"{name}/{tag}/sizes{lv}"] = np.asarray(sizes, dtype=np.int64)
            m = ref.pack_csrk(a, res.perm, res.level_group_sizes)
            out[f"{name}/{tag}/base_row_ptr"] = m.base.row_ptr
            out[f"{name}/{tag}/base_col_idx"] = m.base.col_idx
            out[f"{name}/{tag}/base_vals"] = m.base.vals
            for lv, p in enumerate(m.group_ptrs):
                out[f"{name}/{tag}/ptr{lv}"] = p
            for xs in ("pos", "sgn"):
                x = out[f"{name}/x_{xs}"]
                xp = ref.permute_vector(res.perm, x)
                if k == 2:
                    out[f"{name}/{tag}/y_csr2_{xs}"] = ref.spmv_csr2(m, xp)
                    continue
                out[f"{name}/{tag}/y_csr3_{xs}"] = ref.spmv_csr3(m, xp)
                for d in EMU3_DIMS:
                    y, tr = ref.emulate_gpu_spmv3(m, xp, ref.BlockDims(*d))
                    dt = "x".join(map(str, d))
                    # the serial mapping is bitwise csr3 (kernels.py:224-261)
                    assert np.array_equal(y, out[f"{name}/{tag}/y_csr3_{xs}"])
                    if xs == "pos" and tag == "k3_4_2" and d == (8, 12, 1):
                        out[f"{name}/{tag}/trace_emu3_{dt}"] = np.stack(
                            [tr.row, tr.block, tr.z_lane, tr.y_lane, tr.x_first,
                             tr.x_count, tr.reduction_depth]).astype(np.int32)
                for d in EMU35_DIMS:
                    y, tr = ref.emulate_gpu_spmv35(m, xp, ref.BlockDims(*d))
                    dt = "x".join(map(str, d))
                    if xs == "sgn" or d in EMU35_BOTH:
                        out[f"{name}/{tag}/y_emu35_{dt}_{xs}"] = y
                    if xs == "pos" and tag == "k3_4_2" and d in EMU35_BOTH:
                        out[f"{name}/{tag}/trace_emu35_{dt}"] = np.stack(
                            [tr.row, tr.block, tr.z_lane, tr.y_lane, tr.x_first,
                             tr.x_count, tr.reduction_depth]).astype(np.int32)
    out["names"] = np.array(names)
    path = os.path.join(HERE, "small_cases.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} cases, {os.path.getsize(path) / 1e6:.2f} MB")


def synthetic_tridiagonal(n, seed):
    """pkg/tests/conftest.py:19-29 tridiagonal fixture, rebuilt for fig1."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
    vals = rng.uniform(0.5, 1.5, len(rows))
    return ref.csr_from_arrays(n, n, np.array(rows), np.array(cols), vals)


# ----------------------------------------------------------------------------
# medium / large: digests
# ----------------------------------------------------------------------------

def _build_ref_matrix(spec):
    kind = spec["kind"]
    if kind == "stencil":
        n, rp, ci, v = synthetic.stencil_arrays(spec["shape"], spec["points"],
                                               values=spec.get("values", "laplacian"))
        a = ref.CsrMatrix(n, n, rp, ci, v)
        return a, {"row_ptr": digest(rp, "<u4"), "col_idx": digest(ci, "<u4"),
                   "vals": digest(v, "<f8")}
    rows, cols, vals = synthetic.irregular_triplets(spec["rows"], seed=spec.get("seed", 0))
    a = ref.csr_from_arrays(spec["rows"], spec["rows"], rows, cols, vals)
    return a, {"row_ptr": digest(a.row_ptr, "<u4"), "col_idx": digest(a.col_idx, "<u4"),
               "vals": digest(a.vals, "<f8")}


def run_config(name, spec, targets_list, emu=False, csr_ref=True):
    t0 = time.time()
    a, input_digests = _build_ref_matrix(spec)
    rec = {"spec": spec, "n": a.n_rows, "nnz": a.nnz, "input": input_digests}
    st = ref.compute_stats(a)
    rec["stats"] = {"rdensity": float(st.rdensity).hex(),
                    "variance": float(st.variance).hex(), "max_row_nnz": st.max_row_nnz,
                    "pattern_symmetry": float(st.pattern_symmetry).hex()}
    rec["tune_volta"] = ref.tune_gpu(st, ref.VOLTA).to_dict()
    rec["tune_ampere"] = ref.tune_gpu(st, ref.AMPERE).to_dict()
    x = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
    if csr_ref:
        y_ref = ref.spmv_csr_ref(a, x)
        rec["y_ref"] = digest(y_ref, "<f8")
    rec["runs"] = []
    for entry in targets_list:
        targets, emu_dims = (entry if isinstance(entry, tuple) else (entry, None))
        t1 = time.time()
        res = ref.band_k(a, 3, targets)
        t_band = time.time() - t1
        m = ref.pack_csrk(a, res.perm, res.level_group_sizes)
        xp = ref.permute_vector(res.perm, x)
        y3 = ref.spmv_csr3(m, xp, workers=8)
        run = {
            "targets": list(targets),
            "band_k_seconds": round(t_band, 2),
            "fwd": digest(res.perm.fwd, "<i8"),
            "sizes0": digest(res.level_group_sizes[0], "<i8"),
            "sizes1": digest(res.level_group_sizes[1], "<i8"),
            "n_sr": len(res.level_group_sizes[0]),
            "n_ssr": len(res.level_group_sizes[1]),
            "base_row_ptr": digest(m.base.row_ptr, "<u4"),
            "base_col_idx": digest(m.base.col_idx, "<u4"),
            "base_vals": digest(m.base.vals, "<f8"),
            "sr_ptr": digest(m.sr_ptr, "<u4"),
            "ssr_ptr": digest(m.ssr_ptr, "<u4"),
            "xp": digest(xp, "<f8"),
            "y_csr3": digest(y3, "<f8"),
            "y_csr3_sample": [float(v).hex() for v in y3[:: max(1, a.n_rows // 16)]],
        }
        yu = ref.unpermute_vector(res.perm, y3)
        run["y_csr3_unpermuted"] = digest(yu, "<f8")
        if csr_ref:
            run["max_rel_error_vs_ref"] = ref.max_rel_error(yu, y_ref)
        if emu or emu_dims:
            d = emu_dims or (4, 8, 12)
            dims = ref.BlockDims(*d)
            t2 = time.time()
            y35, _ = ref.emulate_gpu_spmv35(m, xp, dims)
            run["y_emu35_%dx%dx%d" % tuple(d)] = digest(y35, "<f8")
            run["emu35_seconds"] = round(time.time() - t2, 1)
            del y35
        rec["runs"].append(run)
        print(f"  {name} targets {targets}: band_k {t_band:.1f}s", flush=True)
    rec["seconds"] = round(time.time() - t0, 1)
    return rec


MEDIUM = {
    "grid2d_200": ({"kind": "stencil", "shape": [200, 200], "points": 5}, [[8, 8], [4, 8], [16, 16]], True),
    "grid3d7_32": ({"kind": "stencil", "shape": [32, 32, 32], "points": 7}, [[7, 6], [8, 32]], True),
    "grid3d27_20": ({"kind": "stencil", "shape": [20, 20, 20], "points": 27}, [[10, 20], [4, 4]], True),
    "grid3d7_24u": ({"kind": "stencil", "shape": [24, 24, 24], "points": 7, "values": "uniform"}, [[7, 6]], True),
    "irregular_200k": ({"kind": "irregular", "rows": 200_000}, [[14, 9]], True),
    "C1": ({"kind": "stencil", "shape": [1000, 1000], "points": 5}, [[8, 7], [8, 32]], True),
}

LARGE = {
    "C2": ({"kind": "stencil", "shape": [256, 256, 256], "points": 7}, [[7, 6]], False),
    "C3": ({"kind": "stencil", "shape": [192, 192, 192], "points": 27}, [[10, 20]], False),
    "C5": ({"kind": "irregular", "rows": 5_000_000}, [[14, 9]], False),
}


# The B200 profile's picks (paper_2203_05096_b200/data/b200.json through
# tune_gpu) for the benchmarked configs: band_k targets [srs, ssrs] and, for
# the strided order, the block dims whose x lanes the streaming kernel uses.
# C1 [9, 13] dims 2x12x1 (cuda3); C2 [8, 12] 2x12x1 (cuda3); C3 [5, 10]
# 4x8x8 (cuda35); C5 [7, 11] 4x8x12 (cuda3; its strided order pinned too).
B200 = {
    "C1": ({"kind": "stencil", "shape": [1000, 1000], "points": 5}, [([9, 13], (4, 8, 12))]),
    "C2": ({"kind": "stencil", "shape": [256, 256, 256], "points": 7}, [([8, 12], (8, 8, 8))]),
    "C3": ({"kind": "stencil", "shape": [192, 192, 192], "points": 27}, [([5, 10], (4, 8, 8))]),
    "C5": ({"kind": "irregular", "rows": 5_000_000}, [([7, 11], (4, 8, 12))]),
}


def add_b200_runs():
    """Append runs at the B200 profile's targets to the existing entries of
    configs.json (the input / stats digests are already there)."""
    path = os.path.join(HERE, "configs.json")
    with open(path) as fh:
        data = json.load(fh)
    only = sys.argv[2:]
    for name, (spec, runs) in B200.items():
        if only and name not in only:
            continue
        print(f"{name} (b200 targets) ...", flush=True)
        rec = run_config(name, spec, runs, emu=False, csr_ref=False)
        old = data.setdefault(name, rec)
        if old is not rec:
            if old["input"] != rec["input"]:
                raise SystemExit(f"{name}: input digests changed")
            have = {tuple(r["targets"]) for r in old["runs"]}
            old["runs"] += [r for r in rec["runs"] if tuple(r["targets"]) not in have]
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
            fh.write("\n")
    print(f"wrote {path}")


def configs(which):
    path = os.path.join(HERE, "configs.json")
    data = {}
    if os.path.exists(path):
        with open(path) as fh:
            data = json.load(fh)
    table = MEDIUM if which == "medium" else LARGE
    only = sys.argv[2:]
    for name, (spec, targets, emu) in table.items():
        if only and name not in only:
            continue
        print(f"{name} ...", flush=True)
        data[name] = run_config(name, spec, targets, emu=emu,
                                csr_ref=(which == "medium"))
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
            fh.write("\n")
    print(f"wrote {path}")


def mm():
    """Matrix Market ingest (io.py:96-206), writer (209-230) and permutation
    files (278-299) of the reference on the deterministic cases of
    mm_cases.py: digests of the CSR arrays it reads, of the text it writes
    back, and of a permutation file."""
    import io as _io

    sys.path.insert(0, HERE)
    import mm_cases

    out = {}
    for name in mm_cases.CASES:
        t0 = time.time()
        a = ref.io.read_matrix_market(_io.StringIO(mm_cases.mm_text(name)))
        w = _io.StringIO()
        ref.io.write_matrix_market(a, w)
        perm = ref.Permutation.from_forward(mm_cases.perm_of(a.n_rows))
        pf = _io.StringIO()
        ref.io.write_permutation_file(perm, pf)
        out[name] = {"n_rows": a.n_rows, "n_cols": a.n_cols, "nnz": a.nnz,
                     "row_ptr": digest(a.row_ptr, "<u4"), "col_idx": digest(a.col_idx, "<u4"),
                     "vals": digest(a.vals, "<f8"),
                     "written": hashlib.sha256(w.getvalue().encode()).hexdigest(),
                     "perm_file": hashlib.sha256(pf.getvalue().encode()).hexdigest()}
        print(f"{name}: nnz {a.nnz} ({time.time() - t0:.1f}s)", flush=True)
    # the packaged manifest of the paper's 64 matrices, as the reference loads it
    ents = ref.io.load_manifest()
    out["_manifest"] = {"count": len(ents), "entries": hashlib.sha256(
        repr([tuple(e.__dict__.values()) for e in ents]).encode()).hexdigest()}
    path = os.path.join(HERE, "mm.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "small"
    if mode == "small":
        small()
    elif mode in ("medium", "large"):
        configs(mode)
    elif mode == "b200":
        add_b200_runs()
    elif mode == "mm":
        mm()
    else:
        raise SystemExit(f"unknown mode {mode}")
