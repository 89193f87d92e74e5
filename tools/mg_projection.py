"""Multi-GPU partition of the benched CSR-k matrices, and a MODEL of the
N-GPU step time -- not a measurement (every gpurun call has one GPU).

For C2 / C3 (optionally C5) at N = 1, 2, 4, 8 this builds the exact CSR-k
matrix the bench times (the reference's own band_k permutation with the B200
profile's targets, cached in baseline/_cache by `bench.py --impl reference`,
packed by the reference's pack_csrk on the host), then runs the package's
own partition code (dist.partition_by_nnz / footprints / halo_plan /
interior_rows: what DistSpMV and csrk_mg_* use) and reports per rank:
rows, nonzeros, the footprint of x, halo bytes in / out, the interior share
of the rows, and the local algorithmic bytes.

Model of one step at N GPUs (stated assumptions, printed with the result):
  t_comp(g)   = T1 * local_bytes(g) / bytes(N = 1)       (the measured one-GPU
                kernel rate carried over to the rank's own bytes)
  t_xchg(g)   = LAT + max(in_bytes, out_bytes) / BW_NVL  (NCCL send / recv)
  t_step(g)   = max(interior share * t_comp, t_xchg) + boundary share *
                t_comp + 2 * T_LAUNCH                      (interior tiles
                overlap the exchange; boundary tiles after it)
  efficiency  = T1 / (N * max_g t_step(g))
with LAT = 15 us, BW_NVL = 700 GB/s per direction, T_LAUNCH = 3 us.

    python tools/mg_projection.py C2 C3 > profiles/r02_mg_projection.jsonl
"""
from __future__ import annotations

import glob
import importlib.util
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2203_05096_b200 import dist, synthetic  # noqa: E402

LAT_US, BW_NVL, T_LAUNCH_US = 15.0, 700e9, 3.0
TILE = 1536  # the auto plan's tile cost for regular rows
# measured one-GPU kernel times (ms), profiles/SUMMARY_r02.md
T1_MS = {"C2": (0.2549, 0.2754), "C3": (0.3915, 0.4093), "C5": (0.2121, 0.2228)}


def _reference():
    path = os.path.join(REPO, "baseline", "_ref", "csrk", "__init__.py")
    spec = importlib.util.spec_from_file_location(
        "csrk", path, submodule_search_locations=[os.path.dirname(path)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["csrk"] = mod
    spec.loader.exec_module(mod)
    return mod


def build(ref, cfg):
    kind, shape, points = synthetic.CONFIGS[cfg]
    if kind == "stencil":
        n, rp, ci, va = synthetic.stencil_arrays(shape, points)
        a = ref.CsrMatrix(n, n, rp, ci, va)
    else:
        rows, cols, vals = synthetic.irregular_triplets(shape)
        a = ref.csr_from_arrays(shape, shape, rows, cols, vals)
    cache = sorted(glob.glob(os.path.join(REPO, "baseline", "_cache", f"{cfg}_k3_*.npz")))
    if not cache:
        raise SystemExit(f"no cached reference permutation for {cfg}: run "
                         f"`python bench.py --impl reference --config {cfg}` first")
    z = np.load(cache[-1])
    perm = ref.Permutation.from_forward(z["fwd"].astype(np.int64))
    m = ref.pack_csrk(a, perm, [z["sizes0"].tolist(), z["sizes1"].tolist()])
    return m, os.path.basename(cache[-1])


def project(cfg, m, src):
    b = m.base
    rp = np.asarray(b.row_ptr, dtype=np.int64)
    ci = np.asarray(b.col_idx)
    n, nnz = b.n_rows, int(rp[-1])
    vb = 8

    def local_bytes(r0, r1, f0, f1):
        k = int(rp[r1] - rp[r0])
        return k * (vb + 4) + 4 * (r1 - r0 + 1) + vb * (r1 - r0) + vb * (f1 - f0)

    bytes1 = local_bytes(0, n, 0, n)
    out = []
    for world in (1, 2, 4, 8):
        cuts = dist.partition_by_nnz(rp, m.sr_ptr, m.ssr_ptr, world)
        fps = dist.footprints(rp, ci, cuts)
        plan = dist.halo_plan(cuts, fps)
        ranks = []
        for g in range(world):
            r0, r1 = int(cuts[g]), int(cuts[g + 1])
            p0, p1 = int(rp[r0]), int(rp[r1])
            ia, ib = dist.interior_rows(rp[r0:r1 + 1] - p0, ci[p0:p1], r0, r1)
            hin = sum((hi - lo) * vb for s, d, lo, hi in plan if d == g)
            hout = sum((hi - lo) * vb for s, d, lo, hi in plan if s == g)
            lb = local_bytes(r0, r1, int(fps[g][0]), int(fps[g][1]))
            interior_nnz = int(rp[r0 + ib] - rp[r0 + ia]) if ib > ia else 0
            # the true interior set (rows reading only owned columns, not
            # necessarily contiguous), its share at tile granularity (tiles of
            # TILE cost units = nonzeros + rows, as the streaming kernel cuts
            # them), and the halo as the distinct columns read (not the window)
            lrp = rp[r0:r1 + 1]
            nzr = lrp[1:] > lrp[:-1]
            first = np.where(nzr, ci[np.minimum(lrp[:-1], max(nnz - 1, 0))], r0).astype(np.int64)
            last = np.where(nzr, ci[np.maximum(lrp[1:] - 1, 0)], r0).astype(np.int64)
            row_in = (first >= r0) & (last < r1)
            row_nnz = lrp[1:] - lrp[:-1]
            set_nnz = int(row_nnz[row_in].sum())
            cost = np.cumsum(row_nnz + 1)
            tile_of = (cost - 1) // TILE
            n_t = int(tile_of[-1]) + 1 if len(tile_of) else 0
            bad = np.zeros(n_t, dtype=bool)
            np.logical_or.at(bad, tile_of, ~row_in)
            tile_nnz = np.bincount(tile_of, weights=row_nnz, minlength=n_t)
            tiles_nnz = int(tile_nnz[~bad].sum())
            cols = ci[p0:p1]
            outside = cols[(cols < r0) | (cols >= r1)]
            sparse_in = int(np.unique(outside).size) * vb
            ranks.append({"rows": r1 - r0, "nnz": p1 - p0, "footprint": int(fps[g][1] - fps[g][0]),
                          "halo_in_bytes": int(hin), "halo_out_bytes": int(hout),
                          "interior_nnz_share": round(interior_nnz / max(1, p1 - p0), 4),
                          "interior_set_nnz_share": round(set_nnz / max(1, p1 - p0), 4),
                          "interior_tiles_nnz_share": round(tiles_nnz / max(1, p1 - p0), 4),
                          "sparse_halo_in_bytes": sparse_in,
                          "local_bytes": int(lb)})
        rec = {"config": cfg, "n_gpus": world, "n_rows": n, "nnz": nnz, "matrix": src,
               "max_halo_in_MB": round(max(r["halo_in_bytes"] for r in ranks) / 1e6, 3),
               "max_local_bytes_over_ideal": round(max(r["local_bytes"] for r in ranks)
                                                   / (bytes1 / world), 4),
               "min_interior_share": min(r["interior_nnz_share"] for r in ranks),
               "min_interior_tiles_share": min(r["interior_tiles_nnz_share"] for r in ranks),
               "max_sparse_halo_in_MB": round(max(r["sparse_halo_in_bytes"] for r in ranks) / 1e6, 3)}
        for label, t1 in zip(("1965MHz", "power_capped"), T1_MS.get(cfg, (None, None))):
            if t1 is None:
                continue
            t1_us = t1 * 1e3
            steps = []
            for r in ranks:
                tc = t1_us * r["local_bytes"] / bytes1
                tx = (LAT_US + max(r["halo_in_bytes"], r["halo_out_bytes"]) / BW_NVL * 1e6
                      if world > 1 else 0.0)
                sh = r["interior_nnz_share"] if world > 1 else 1.0
                launch = 2 * T_LAUNCH_US if world > 1 else 0.0
                steps.append(max(sh * tc, tx) + (1 - sh) * tc + launch)
            tn = max(steps)
            rec[f"model_{label}"] = {"t1_us": round(t1_us, 1), "tN_us": round(tn, 1),
                                     "efficiency": round(t1_us / (world * tn), 3)}
            # the same with interior TILES (a tile list per launch) and the
            # sparse halo (distinct columns only)
            steps2 = []
            for r in ranks:
                tc = t1_us * r["local_bytes"] / bytes1
                tx = (LAT_US + r["sparse_halo_in_bytes"] / BW_NVL * 1e6 if world > 1 else 0.0)
                sh = r["interior_tiles_nnz_share"] if world > 1 else 1.0
                launch = 2 * T_LAUNCH_US if world > 1 else 0.0
                steps2.append(max(sh * tc, tx) + (1 - sh) * tc + launch)
            tn2 = max(steps2)
            rec[f"model_tiles_sparse_{label}"] = {"tN_us": round(tn2, 1),
                                                  "efficiency": round(t1_us / (world * tn2), 3)}
        rec["assumptions"] = (f"model, not a measurement: LAT {LAT_US} us, NVLink {BW_NVL / 1e9:.0f} "
                              f"GB/s per direction, {T_LAUNCH_US} us per extra launch, one-GPU "
                              f"rate carried over per rank")
        rec["ranks"] = ranks
        out.append(rec)
        print(json.dumps(rec), flush=True)
    return out


def main():
    ref = _reference()
    for cfg in sys.argv[1:] or ["C2", "C3"]:
        m, src = build(ref, cfg)
        project(cfg, m, src)


if __name__ == "__main__":
    main()
