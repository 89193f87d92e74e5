"""Measure the B200 tuning data for the CSR-k model (run on a B200).

For a family of synthetic matrices spanning row densities 3..40 (grid
stencils and irregular random-row-length matrices, all larger than L2), this
times the streaming kernel for every (SSRS, SRS) pair of the B200 candidate
grid (paper_2203_05096_b200.tuning.b200_candidate_grid), in the serial order
and in the strided order with nx in {2, 4, 8, 16}, using CUDA events (median
of 10 launches after warm-up).  Band-k + device pack run once per pair.

Writes gpurun_out/fit_b200_raw.json; tools/make_b200_profile.py turns it
into paper_2203_05096_b200/data/b200.json with fit_log_model (the
reference's tuning.py:444-468 procedure).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402

FAMILY = [
    ("stencil2d5", lambda: synthetic.stencil_arrays((3000, 3000), 5)),
    ("stencil3d7", lambda: synthetic.stencil_arrays((160, 160, 160), 7)),
    ("stencil2d9", lambda: synthetic.stencil_arrays((2000, 2000), 9)),
    ("stencil3d27", lambda: synthetic.stencil_arrays((100, 100, 100), 27)),
    ("stencil3d27_l", lambda: synthetic.stencil_arrays((160, 160, 160), 27)),
    ("irreg_l5", lambda: _irregular(6_000_000, 5)),
    ("irreg_l11", lambda: _irregular(3_000_000, 11)),
    ("irreg_l19", lambda: _irregular(2_000_000, 19)),
    ("irreg_l39", lambda: _irregular(1_000_000, 39)),
    ("irreg_l79", lambda: _irregular(500_000, 79)),
]
NX = (2, 4, 8, 16)


def _irregular(n, max_len):
    r, c, v = synthetic.irregular_triplets(n, seed=0, max_len=max_len)
    a = ck.csr_from_arrays(n, n, r, c, v)
    return a.n_rows, a.row_ptr, a.col_idx, a.vals


def time_kernel(m, xd, yd, dims, variant, reps=10):
    for _ in range(3):
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    return float(np.median(times))


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fit_b200_raw.json"
    only = set(sys.argv[2:])
    results = {}
    if os.path.exists(out_path):
        with open(out_path) as fh:
            results = json.load(fh)
    for name, make in FAMILY:
        if only and name not in only:
            continue
        t0 = time.time()
        n, rp, ci, va = make()
        a = ck.CsrMatrix(n, n, rp, ci, va, _trusted=True)
        st = ck.compute_stats(a)
        x = np.random.default_rng(0).uniform(-1, 1, n)
        rec = {"n": n, "nnz": a.nnz, "rdensity": st.rdensity, "variance": st.variance,
               "max_row_nnz": st.max_row_nnz, "runs": []}
        for ssrs, srs in ck.b200_candidate_grid():
            res = ck.band_k(a, 3, [srs, ssrs])
            m = ck.pack_csrk(a, res.perm, res.level_group_sizes, download=False)
            xd = torch.from_numpy(x[res.perm.inv]).cuda()
            yd = torch.empty(n, dtype=torch.float64, device="cuda")
            run = {"ssrs": ssrs, "srs": srs, "n_sr": len(res.level_group_sizes[0]),
                   "n_ssr": len(res.level_group_sizes[1]),
                   "serial_ms": time_kernel(m, xd, yd, None, "serial")}
            for nx in NX:
                run[f"strided{nx}_ms"] = time_kernel(m, xd, yd, ck.BlockDims(nx, 1, 1),
                                                     "strided")
            rec["runs"].append(run)
            del m, xd, yd
            torch.cuda.empty_cache()
        rec["seconds"] = round(time.time() - t0, 1)
        results[name] = rec
        best = min(rec["runs"], key=lambda r: min(v for k, v in r.items() if k.endswith("_ms")))
        print(f"{name}: rd={st.rdensity:.2f} nnz={a.nnz} best={best} ({rec['seconds']}s)",
              flush=True)
        os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
        with open(out_path, "w") as fh:
            json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
