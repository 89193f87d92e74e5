"""Fit the B200 CSR-k model from tools/fit_b200.py measurements.

For every matrix of the family: the fastest (variant, SSRS, SRS) of the grid.
Then, as the paper does for Volta / Ampere with the
reference's fit_log_model (tuning.py:444-468):

  ssrs_coeff, srs_coeff  least-squares fits of size = a - b ln(rdensity)
                         over the per-matrix optima;
  case table             the paper's four row-density intervals; dims.x of
                         each = the lane count that won most often inside it
                         (the strided order's nx), no size adjustments
                         (the fitted formulas already are B200 optima);
  serial threshold       the largest rdensity at which the serial order won.

Writes paper_2203_05096_b200/data/b200.json (profile keys plus a "fit"
record of the measurements it came from).

    python tools/make_b200_profile.py gpurun_out/fit_b200_raw.json
"""

from __future__ import annotations

import collections
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_05096_b200 import tuning as T  # noqa: E402
from paper_2203_05096_b200.kernels import BlockDims  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2203_05096_b200", "data", "b200.json")
UPPERS = (8.0, 16.0, 32.0, None)
DEFAULT_DIMS = ((8, 12, 1), (4, 8, 12), (8, 8, 8), (16, 8, 4))


def best_of(rec):
    best = None
    for run in rec["runs"]:
        for key, ms in run.items():
            if not key.endswith("_ms"):
                continue
            variant = key[:-3]
            nx = 0 if variant == "serial" else int(variant.replace("strided", ""))
            cand = (ms, run["ssrs"], run["srs"], nx)
            if best is None or cand < best:
                best = cand
    return best


def main(path):
    with open(path) as fh:
        data = json.load(fh)
    rows = []
    for name, rec in sorted(data.items(), key=lambda kv: kv[1]["rdensity"]):
        ms, ssrs, srs, nx = best_of(rec)
        serial_ms = min(r["serial_ms"] for r in rec["runs"])
        rows.append({"matrix": name, "rdensity": rec["rdensity"], "variance": rec["variance"],
                     "nnz": rec["nnz"], "best_ms": ms, "ssrs": ssrs, "srs": srs,
                     "nx": nx, "serial_best_ms": serial_ms,
                     "gflops": round(2 * rec["nnz"] / (ms * 1e-3) / 1e9, 1)})
    ssrs_coeff = T.fit_log_model([(r["rdensity"], r["ssrs"]) for r in rows])
    srs_coeff = T.fit_log_model([(r["rdensity"], r["srs"]) for r in rows])
    serial_rd = [r["rdensity"] for r in rows if r["nx"] == 0]
    threshold = max(serial_rd) if serial_rd else 0.0
    cases = []
    lo = 0.0
    for upper, default in zip(UPPERS, DEFAULT_DIMS):
        inside = [r for r in rows if r["rdensity"] > lo and (upper is None or r["rdensity"] <= upper)
                  and r["nx"] > 0]
        if inside:
            nx = collections.Counter(r["nx"] for r in inside).most_common(1)[0][0]
            dims = BlockDims(nx, default[1], max(1, default[2]) if nx * default[1] * default[2]
                             <= 1024 else 1)
        else:
            dims = BlockDims(*default)
        cases.append(T.CaseRule(upper, dims))
        lo = upper if upper is not None else lo
    prof = T.DeviceProfile(name="b200", ssrs_coeff=tuple(round(v, 4) for v in ssrs_coeff),
                           srs_coeff=tuple(round(v, 4) for v in srs_coeff),
                           case_table=tuple(cases),
                           serial_inner_threshold=float(math.floor(threshold * 100) / 100))
    d = T.profile_to_dict(prof)
    d["fit"] = {"source": "tools/fit_b200.py on one B200 (CUDA-event medians)",
                "candidates": [list(c) for c in T.b200_candidate_grid()],
                "per_matrix_optima": rows}
    with open(OUT, "w") as fh:
        json.dump(d, fh, indent=2)
        fh.write("\n")
    print(json.dumps({k: d[k] for k in ("ssrs_coeff", "srs_coeff", "serial_inner_threshold")}))
    for r in rows:
        print(r)
    assert T.load_profile(OUT) == prof


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fit_b200_raw.json")
