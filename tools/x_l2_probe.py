"""x-isolated L2 / L1 hit rates ("a gather-only kernel
variant to isolate x"), run on a B200 under ncu.

For each config: the CSR-k matrix as bench.py builds it (B200 model, device
Band-k), then csrk_probe_gather mode 0 (col_idx stream only) and mode 1
(col_idx + x gathers), each launched twice (first warm, second profiled).
Run as

  ncu --clock-control none -k regex:gather_probe --metrics <M> --csv \
      --log-file gpurun_out/x_l2.csv python tools/x_l2_probe.py C1 C2 C3 C5

and summarise with ``python tools/x_l2_probe.py --summarise gpurun_out/x_l2.csv``:
x's own sector hits / lookups = (mode 1 - mode 0) over both counters.
Without ncu it also prints each probe's event time (bare gather rate).
"""

from __future__ import annotations

import csv
import json
import os
import sys

METRICS = ("lts__t_sectors_srcunit_tex_op_read.sum,"
           "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,"
           "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,"
           "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,"
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,"
           "lts__t_sectors_srcunit_tex_op_read_evict_normal.sum,"
           "lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_hit.sum,"
           "lts__t_sectors_srcunit_tex_op_read_evict_first.sum,"
           "lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_hit.sum,"
           "lts__t_sector_hit_rate.pct,"
           "dram__bytes_read.sum,gpu__time_duration.sum")


def run(configs):
    import numpy as np
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2203_05096_b200 import _native as nat

    for cfg in configs:
        a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
        dev = m.device()
        xd = torch.from_numpy(xp).to("cuda")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        for mode in (0, 1):
            ts = []
            for rep in range(4):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                nat.call("csrk_probe_gather", dev.ptr, mode, xd.data_ptr(), out.data_ptr(), s)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            print(json.dumps({"config": cfg, "mode": mode, "nnz": a.nnz,
                              "ms_median": float(np.median(ts[1:])),
                              "gathers_per_s": a.nnz / (float(np.median(ts[1:])) * 1e-3)
                              if mode else None}), flush=True)
        # the SpMV itself (same matrix and x, the bench's order), twice: its x
        # gathers are the only evict-normal reads (the matrix streams with
        # L2 evict_first TMA copies), so ncu's evict_normal sector counters
        # of this launch are x's own hit rate inside the real kernel
        import paper_2203_05096_b200 as ck
        variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
        yd = torch.empty_like(xd)
        for _ in range(2):
            ck.spmv_device(m, xd, yd, dims=params.block_dims, variant=variant)
        torch.cuda.synchronize()
        del m, dev, xd, yd
        torch.cuda.empty_cache()


def summarise(path, configs=("C1", "C2", "C3", "C5")):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    by = {}
    for r in rows:
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        by.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})[r["Metric Name"]] = v
    launches = [by[k] for k in sorted(by)]
    out = []
    per = 10  # per config: probe mode 0 x4, mode 1 x4, SpMV x2
    for ci in range(len(launches) // per):
        L = launches[ci * per:(ci + 1) * per]
        m0, m1, sp = L[3], L[7], L[9]
        d = {k: m1[k] - m0[k] for k in m1 if k in m0 and k != "kernel"}
        en = "lts__t_sectors_srcunit_tex_op_read_evict_normal"
        rec = {"config": configs[ci] if ci < len(configs) else ci,
               "probe_x_l2_hit_rate": d[en + "_lookup_hit.sum"] / d[en + ".sum"],
               "probe_x_l1_hit_rate":
                   d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum"] /
                   d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"],
               "probe_x_l2_sectors": d[en + ".sum"],
               "probe_x_requests": d["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"],
               "probe_x_dram_bytes": d["dram__bytes_read.sum"],
               "spmv_kernel": sp["kernel"][:40],
               "spmv_x_l2_hit_rate": sp[en + "_lookup_hit.sum"] / sp[en + ".sum"]
               if sp.get(en + ".sum") else None,
               "spmv_x_l1_hit_rate":
                   sp["l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum"] /
                   sp["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
                   if sp.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") else None,
               "spmv_x_l2_sectors": sp.get(en + ".sum"),
               "spmv_whole_l2_hit_pct": sp.get("lts__t_sector_hit_rate.pct"),
               "spmv_dram_read_bytes": sp.get("dram__bytes_read.sum"),
               "probe_mode0_time": m0["gpu__time_duration.sum"],
               "probe_mode1_time": m1["gpu__time_duration.sum"],
               "spmv_time": sp["gpu__time_duration.sum"]}
        out.append(rec)
        print(json.dumps(rec))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--summarise":
        summarise(sys.argv[2])
    elif len(sys.argv) > 1 and sys.argv[1] == "--metrics":
        print(METRICS)
    else:
        run(sys.argv[1:] or ["C1", "C2", "C3", "C5"])
