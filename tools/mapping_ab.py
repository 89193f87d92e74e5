"""CSR-k mapping A/B and held-out model table (run on a B200).

VERDICT r01 "Next round" 7: does the paper's super-super-row -> CTA mapping
pay on B200, and does the fitted B200 model pick good group sizes on
matrices it was not fitted on (C1, C2, C3, C5 are not in tools/fit_b200.py's
family)?

For every config and every (SSRS, SRS) of the B200 candidate grid (plus the
Volta / Ampere / B200 model picks), Band-k + pack run on the device once,
then (fp64, CUDA events, median of 20 launches; C1 with an L2 flush before
every launch):

  rows     the streaming kernel with tile cuts on rows (cut mode 1)
  groups   the streaming kernel with tile cuts on super-super-row
           boundaries only (cut mode 2, the paper's block <-> SSR mapping
           coarsened to a tile), best over tile costs 2048 / 3072 / 4096
  listing  for the three model picks: the paper's literal mapping (PAPER
           Listing 3 for GPU3 picks, Listing 4 for GPU35 picks, grid = n_SSR,
           block = the profile's dims; csrk_spmv_listing3/4 without trace)

All variants of one matrix are checked bitwise against the first.  Writes
gpurun_out/mapping_ab.json and prints one JSON line per measurement.
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
from paper_2203_05096_b200 import _native as nat  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402

GRID = os.environ.get("AB_GRID", "1") == "1"
GROUP_TILES = (2048, 3072, 4096)
FLUSH = torch.empty(64 << 20, dtype=torch.float64, device="cuda")


def median_ms(fn, flush, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            FLUSH.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def order_of(params):
    v = params.kernel_variant.value
    if v in ("cuda35", "gpu35-emu"):
        return "strided", params.block_dims
    return "serial", params.block_dims


def main():
    configs = sys.argv[1:] or ["C1", "C2", "C3", "C5"]
    out = []
    profiles = {"b200": ck.b200_profile(), "volta": ck.VOLTA, "ampere": ck.AMPERE}
    for cfg in configs:
        t0 = time.time()
        n, rp, ci, va = synthetic.config_arrays(cfg)
        a = ck.CsrMatrix(n, n, rp, ci, va, _trusted=True)
        stats = ck.compute_stats(a)
        picks = {name: ck.tune_gpu(stats, p) for name, p in profiles.items()}
        model_order, model_dims = order_of(picks["b200"])
        pairs = {}
        for name, p in picks.items():
            pairs.setdefault((p.ssrs, p.srs), []).append(name)
        if GRID:
            for pr in ck.b200_candidate_grid():
                pairs.setdefault(pr, [])
        x = synthetic.config_x(n)
        nb = spmv_bytes(n, n, a.nnz, 8)
        flush = nb < 4 * 126e6
        for (ssrs, srs), names in sorted(pairs.items()):
            tb = time.time()
            res = ck.band_k(a, 3, [srs, ssrs])
            m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
            t_build = time.time() - tb
            xp = ck.permute_vector(res.perm, x)
            xd = torch.from_numpy(xp).to("cuda")
            yd = torch.empty(n, dtype=torch.float64, device="cuda")
            dev = m.device()
            orders = [(model_order, model_dims, "b200")]
            for name in names:
                o, d = order_of(picks[name])
                if (o, d.x if o == "strided" else 0) != (model_order, model_dims.x if model_order == "strided" else 0):
                    orders.append((o, d, name))
            want = None
            for order, dims, oname in orders:
                def run():
                    ck.spmv_device(m, xd, yd, dims=dims, variant=order)
                rec = {"config": cfg, "ssrs": ssrs, "srs": srs, "picked_by": names,
                       "order": order, "nx": dims.x if order == "strided" else 0,
                       "order_of": oname, "n_sr": m.num_super_rows, "n_ssr": m.num_ssr,
                       "band_k_s": round(t_build, 2), "l2_flush": flush}
                dev.set_plan(0, 0, 0)
                dev.set_cut_mode(1)
                ms = median_ms(run, flush)
                if want is None:
                    want = yd.clone()
                rec["rows_ms"] = round(ms, 4)
                rec["rows_bitwise"] = bool(torch.equal(yd, want))
                best = None
                for tc in GROUP_TILES:
                    dev.set_cut_mode(2)
                    try:
                        dev.set_plan(tc, 0, 0)
                    except ValueError:
                        continue
                    # a group larger than the stage runs its tile from global
                    # memory ("direct" mode, reachable only with cut mode 2):
                    # one timed trial, skipped when it is 3x the row-cut time
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run()
                    e1.record()
                    e1.synchronize()
                    if e0.elapsed_time(e1) > 3 * ms + 0.05:
                        rec.setdefault("groups_skipped_tiles", []).append(
                            [tc, round(e0.elapsed_time(e1), 3)])
                        continue
                    ms_g = median_ms(run, flush)
                    same = bool(torch.equal(yd, want))
                    pl = dev.plan()
                    if best is None or ms_g < best[0]:
                        best = (ms_g, tc, same, pl.get("group_aligned"), pl.get("n_tiles"))
                dev.set_plan(0, 0, 0)
                dev.set_cut_mode(0)
                if best:
                    rec.update(groups_ms=round(best[0], 4), groups_tile=best[1],
                               groups_bitwise=best[2], groups_aligned=best[3],
                               groups_tiles=best[4])
                ms_auto = median_ms(run, flush)
                rec["auto_ms"] = round(ms_auto, 4)
                rec["auto_gbs"] = round(nb / (ms_auto * 1e-3) / 1e9, 1)
                rec["auto_plan"] = {k: v for k, v in dev.plan().items()
                                    if k in ("tile_cost", "group_aligned", "n_tiles",
                                             "gather_first", "ctas_per_sm")}
                if oname == "b200":
                    # the paper's literal launch mapping (grid = n_SSR, block =
                    # the picking profile's dims) for each profile that picked
                    # this pair, in that profile's order
                    for name in names:
                        o, pdims = order_of(picks[name])
                        if o == "serial":
                            fn = lambda: nat.call("csrk_spmv_listing3", dev.ptr, pdims.x,
                                                  pdims.y, xd.data_ptr(), yd.data_ptr(), None,
                                                  torch.cuda.current_stream().cuda_stream)
                        else:
                            fn = lambda: nat.call("csrk_spmv_listing4", dev.ptr, pdims.x,
                                                  pdims.y, pdims.z, xd.data_ptr(),
                                                  yd.data_ptr(), None,
                                                  torch.cuda.current_stream().cuda_stream)
                        ms_l = median_ms(fn, flush)
                        rec[f"listing_{name}_ms"] = round(ms_l, 4)
                        rec[f"listing_{name}_dims"] = [pdims.x, pdims.y, pdims.z]
                        rec[f"listing_{name}_order"] = o
                print(json.dumps(rec), flush=True)
                out.append(rec)
            del m, dev, xd, yd
            torch.cuda.empty_cache()
        print(f"[ab] {cfg} done in {time.time() - t0:.0f}s", file=sys.stderr, flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        with open("gpurun_out/mapping_ab.json", "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
