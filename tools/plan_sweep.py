"""Sweep the streaming kernel's tile plan (tile cost x ring depth) on B200.

For the given configs, builds the CSR-k matrix once and times the kernel
(CUDA events, median of 20 launches) for every plan in the grid, in fp64 and
fp32, with the tuned variant.  Prints one JSON line per (config, dtype, plan)
and writes gpurun_out/plan_sweep.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402

TILES = tuple(int(t) for t in os.environ.get('SWEEP_TILES', '1024,1280,1536,1792,2048,2560,3072').split(','))
STAGES = tuple(int(t) for t in os.environ.get('SWEEP_STAGES', '2,3').split(','))
GATHER = tuple(int(t) for t in os.environ.get('SWEEP_GATHER', '0,1').split(','))
DTYPES = tuple(getattr(torch, d) for d in os.environ.get('SWEEP_DTYPES', 'float64,float32').split(','))
VARIANTS = os.environ.get('SWEEP_VARIANTS', '')
CTAS_LIST = tuple(int(t) for t in os.environ.get('SWEEP_CTAS', '3').split(','))
LAYOUTS = tuple(int(t) for t in os.environ.get('SWEEP_LAYOUT', '0').split(','))


FLUSH = None
if os.environ.get("SWEEP_FLUSH") == "1":  # write 256 MB (> L2) before every timed launch
    FLUSH = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def median_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if FLUSH is not None:
            FLUSH.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    configs = sys.argv[1:] or ["C2", "C3", "C5"]
    out = []
    for cfg in configs:
        if cfg.startswith("PL"):  # power-law rows, 2 M rows, max row length PL<len>
            from powerlaw_probe import build_powerlaw
            a, m, _, params = build_powerlaw(2_000_000, int(cfg[2:]))
            xp = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
        else:
            a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
        n, nnz = a.n_rows, a.nnz
        variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
        dev = m.device()
        for dtype in DTYPES:
            xd = torch.from_numpy(xp).to("cuda", dtype)
            yd = torch.empty(n, dtype=dtype, device="cuda")
            vb = 8 if dtype == torch.float64 else 4
            variants = VARIANTS.split(',') if VARIANTS else sorted({variant, "serial"})
            nx_list = [int(v) for v in os.environ.get("SWEEP_NX", "").split(",") if v]
            if nx_list:  # strided with explicit lane counts: "strided:<nx>"
                variants = [v for v in variants if v != "strided"] + \
                    [f"strided:{k}" for k in nx_list]
            for variant_i in variants:
                dims = params.block_dims
                if variant_i.startswith("strided:"):
                    variant_i, k = variant_i.split(":")
                    dims = ck.BlockDims(int(k), 1, 1)
                dev.set_plan(0, 0, 0)
                dev.set_schedule(0, 0)
                dev.set_cut_mode(0)
                want = ck.spmv_device(m, xd, yd, dims=dims, variant=variant_i).clone()
                for g, CTAS, LAY in [(g, c, la) for g in (GATHER if vb == 8 else (0,))
                                     for c in CTAS_LIST for la in LAYOUTS]:
                  dev.set_schedule(g, CTAS)
                  dev.set_cut_mode(LAY)
                  for t in TILES:
                    for s in STAGES:
                        try:
                            dev.set_plan(t, 0, s)
                        except ValueError:
                            continue
                        ms = median_ms(lambda: ck.spmv_device(m, xd, yd, dims=dims,
                                                              variant=variant_i))
                        same = bool(torch.equal(yd, want))
                        gbs = spmv_bytes(n, n, nnz, vb) / (ms * 1e-3) / 1e9
                        rec = {"config": cfg, "dtype": str(dtype)[6:], "variant": variant_i,
                               "nx": dims.x if variant_i == "strided" else 0,
                               "gather": g, "ctas": CTAS, "cut_mode": LAY, "tile_cost": t, "stages": s, "ms": round(ms, 4),
                               "gbs": round(gbs, 1), "bitwise_equal": same}
                        print(json.dumps(rec), flush=True)
                        out.append(rec)
            dev.set_plan(0, 0, 0)
            dev.set_schedule(2, 0)
            dev.set_cut_mode(0)
        del m, dev
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/plan_sweep.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
