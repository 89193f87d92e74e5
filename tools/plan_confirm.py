"""Confirm a plan (tile cost, stages, CTAs/SM) with the bench's own timing:
K back-to-back launches between two events, after warm-up, interleaved with
the auto plan, several rounds; bitwise check against the auto plan's y.

    python tools/plan_confirm.py C3 1536 3 3 [--fp32]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def main():
    cfg, tile, stages, ctas = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    f32 = "--fp32" in sys.argv
    if cfg.startswith("PL"):  # power-law rows capped at int(cfg[2:]) (tools/powerlaw_probe.py)
        from powerlaw_probe import build_powerlaw
        a, m, _, params = build_powerlaw(2_000_000, int(cfg[2:]))
        xp = np.random.default_rng(0).uniform(-1.0, 1.0, a.n_rows)
    else:
        a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    dims = params.block_dims
    dt = torch.float32 if f32 else torch.float64
    xd = torch.from_numpy(xp).to("cuda", dt)
    yd = torch.empty(a.n_rows, dtype=dt, device="cuda")
    dev = m.device()
    nb = spmv_bytes(a.n_rows, a.n_rows, a.nnz, 4 if f32 else 8)

    def timed(k=50):
        for _ in range(5):
            ck.spmv_device(m, xd, yd, dims=dims, variant=variant)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            ck.spmv_device(m, xd, yd, dims=dims, variant=variant)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    dev.set_plan(0, 0, 0)
    dev.set_schedule(2, 0)
    timed()
    want = yd.clone()
    auto_plan = dev.plan()
    res = {"auto": [], "plan": []}
    for _ in range(4):
        dev.set_plan(0, 0, 0)
        dev.set_schedule(2, 0)
        res["auto"].append(timed())
        dev.set_plan(tile, 0, stages)
        dev.set_schedule(2, ctas)
        res["plan"].append(timed())
        assert torch.equal(yd, want)
    out = {"config": cfg, "f32": f32, "variant": variant, "nx": dims.x,
           "auto_plan": {k: auto_plan.get(k) for k in ("tile_cost", "stages", "ctas_per_sm",
                                                       "gather_first", "n_tiles")},
           "plan": [tile, stages, ctas],
           "auto_ms": [round(v, 4) for v in res["auto"]],
           "plan_ms": [round(v, 4) for v in res["plan"]],
           "auto_frac": round(nb / (min(res["auto"]) * 1e-3) / 1e9 / 6464.3, 4),
           "plan_frac": round(nb / (min(res["plan"]) * 1e-3) / 1e9 / 6464.3, 4)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
