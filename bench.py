#!/usr/bin/env python
"""Benchmark of the CSR-k SpMV hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--fp32]

Workload (N = 1): BASELINE.json configs[1], the 3D 7-point Laplacian on a
256^3 grid (16.8 M rows, 117 M nonzeros), fp64, CSR-k with k = 3 built by
native Band-k with the model's (SSRS, SRS).  One "step" = one SpMV of the
whole matrix.  Inputs (1.74 GB per SpMV) are larger than the 126 MB L2, so
no flush is needed between steps.

  value      kernel-only GFLOP/s, x / y resident in HBM, CUDA events over K
             back-to-back launches on the launching stream (max over ranks)
  e2e        same metric through the public drop-in call spmv_csr3(m, x)
             with pinned host x / y: H2D of x, kernel, D2H of y every step
  roofline   algorithmic bytes (vals + col_idx + row_ptr + x + y, SURVEY.md
             §8(d)) per launch / measured launch time, against the measured
             HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the reference's CSR-3 algorithm restated in C + OpenMP
             (oracle/, kind "port"), all host cores, bounded sample
  parity     the timed launch's y against the oracle: bitwise in fp64,
             1e-5 of |A||x| in fp32 (the run fails otherwise)

N > 1 (one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run): the SAME matrix as the N = 1 line, its
super-super-rows split across ranks by nonzeros (paper_2203_05096_b200.dist
DistSpMV), each rank holding its rows and a footprint-sized x; every step
posts the x halo over NCCL, computes the interior tiles while it is in
flight, then the boundary tiles (strong scaling; rank 0 also times the whole
matrix on one GPU and prints T1 / (N T_N)).  --config C4: the CG loop on
z-slabs.

``--impl reference`` times the UNMODIFIED reference package (baseline/_ref,
pip-installed from /root/reference/pkg): its own spmv_csr3 with
workers=os.cpu_count() on the CSR-k matrix its own band_k / pack_csrk built
(same config, same B200-model group sizes), on the host cores; no module of
this repo's package and none of its .so files are loaded on that arm.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_TEXT = {
    "C1": "2D 5-point Laplacian 1000x1000 fp64 CSR-k k=3",
    "C2": "3D 7-point Laplacian 256^3 fp64 CSR-k k=3 on 1 B200",
    "C3": "3D 27-point stencil 192^3 fp64 CSR-k k=3",
    "C5": "irregular random-row-length matrix, 5M rows, fp64 CSR-k k=3",
}
METRIC = "SpMV GFLOP/s and achieved HBM GB/s (% of peak) at 1/2/4/8 B200 vs host CPU"


def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi SM clock / throttle-reason samples during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thread = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=10)

    def load_until(self, step, sync, n=3, max_s=3.0):
        """Keep the GPU under the timed workload (untimed) until the sampler
        holds `n` samples, so a short timed region still has clock samples
        taken under the same load right before and during it."""
        have = len(self.samples)
        t0 = time.perf_counter()
        while len(self.samples) < have + n and time.perf_counter() - t0 < max_s:
            for _ in range(8):
                step()
            sync()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_matrix(cfg: str, log):
    """Host CSR of the config, tuned sizes, native Band-k, device pack."""
    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200 import synthetic

    t0 = time.perf_counter()
    n, rp, ci, va = synthetic.config_arrays(cfg)
    a = ck.CsrMatrix(n, n, rp, ci, va, _trusted=True)
    t_gen = time.perf_counter() - t0
    stats = ck.compute_stats(a)
    params = ck.tune_gpu(stats, ck.b200_profile())
    t0 = time.perf_counter()
    res = ck.band_k(a, 3, [params.srs, params.ssrs])
    t_band = time.perf_counter() - t0
    t0 = time.perf_counter()
    m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
    t_pack = time.perf_counter() - t0
    log(f"[bench] {cfg}: n={n} nnz={a.nnz} gen {t_gen:.1f}s band_k {t_band:.1f}s "
        f"pack {t_pack:.1f}s sizes ssrs={params.ssrs} srs={params.srs} "
        f"n_sr={m.num_super_rows} n_ssr={m.num_ssr} variant={params.kernel_variant.value}")
    x = synthetic.config_x(n)
    xp = ck.permute_vector(res.perm, x)
    return a, m, xp, params, {"gen_s": t_gen, "band_k_s": t_band, "pack_s": t_pack}


def cpu_baseline(m, xp, budget_s=10.0, threads=None):
    """Time the oracle's CSR-3 (C + OpenMP restatement of kernels.py:209-221)
    on the host cores: repeat whole-matrix SpMVs for ~budget_s seconds."""
    from oracle import oracle as O

    threads = threads or (os.cpu_count() or 1)
    rows = O.csr3_group_rows(m.sr_ptr, m.ssr_ptr)
    b = m.base
    O.spmv_grouped(rows, b.row_ptr, b.col_idx, b.vals, xp, threads)  # warm-up
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        y = O.spmv_grouped(rows, b.row_ptr, b.col_idx, b.vals, xp, threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or len(times) >= 5000:
            break
    mean = sum(times) / len(times)
    return {"value": round(2.0 * b.nnz / mean / 1e9, 3), "unit": "GFLOP/s",
            "cores": int(threads), "kind": "port",
            "sample": f"{len(times)} full SpMVs of the same CSR-k matrix "
                      f"(oracle/csrk_oracle.c oracle_spmv_grouped, OpenMP static chunks "
                      f"over super-super-rows), mean {mean * 1e3:.1f} ms"}, y


def oracle_y(m, xp, variant, nx, threads=None):
    """The oracle's y for the timed order (test infrastructure: the checker
    of the bench's own output, never the thing measured)."""
    from oracle import oracle as O

    b = m.base
    if variant == "strided":
        return O.spmv_strided(b.row_ptr, b.col_idx, b.vals, xp, nx)
    rows = O.csr3_group_rows(m.sr_ptr, m.ssr_ptr)
    return O.spmv_grouped(rows, b.row_ptr, b.col_idx, b.vals, xp, threads or os.cpu_count())


def parity_of(y_dev, want, m, xp, f32):
    """Bitwise for fp64; for fp32 |y - y64| <= 1e-5 (|A||x|)_i per row
    (north_star's tolerance)."""
    from oracle import oracle as O

    y_dev = np.asarray(y_dev, dtype=np.float64)
    diff = np.abs(y_dev - want)
    if not f32:
        ok = bool(np.array_equal(y_dev, want))
        return {"kind": "bitwise", "ok": ok, "max_abs_diff": float(diff.max()) if diff.size else 0.0,
                "against": "oracle/csrk_oracle.c (pinned to the reference's goldens) on the "
                           "same CSR-k matrix and x"}
    b = m.base
    scale = O.abs_row_dot(b.row_ptr, b.col_idx, b.vals, xp)
    worst = float(np.max(diff / np.maximum(scale, 1e-300))) if diff.size else 0.0
    return {"kind": "scaled", "tolerance": 1e-5, "ok": bool(worst <= 1e-5),
            "max_scaled_error": worst,
            "against": "oracle/csrk_oracle.c fp64 y on the same CSR-k matrix and x"}


def run_ours(args, log):
    import torch

    import paper_2203_05096_b200 as ck
    from paper_2203_05096_b200.bench import spmv_bytes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or (os.environ.get("CSRK_DIST") == "1" and "RANK" in os.environ):
        from paper_2203_05096_b200 import dist
        return dist.bench_main(args, log, sampler=ClockSampler, peak=measured_peak(),
                               oracle_check=oracle_y)
    torch.cuda.set_device(0)
    a, m, xp, params, build_t = build_matrix(args.config, log)
    n, nnz = a.n_rows, a.nnz
    f32 = args.fp32
    dtype = torch.float32 if f32 else torch.float64
    vbytes = 4 if f32 else 8
    dims = params.block_dims
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    xd = torch.from_numpy(xp).to("cuda", dtype)
    yd = torch.empty(n, dtype=dtype, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    algo_bytes = spmv_bytes(n, n, nnz, vbytes)
    # Inputs smaller than 4x the 126 MB L2 (C1: 80 MB) would be served from
    # L2 by back-to-back launches on one copy.  The timed steps rotate
    # instead through R resident replicas of the matrix, x and y (R x the
    # algorithmic bytes >= 4 x L2: each step reads its replica cold from
    # HBM -- "inputs larger than L2"), back to back like the larger configs.
    # The single launch after a 512 MB L2 flush (write, then a read-only pass
    # so the L2 holds no dirty lines), each with its own events, is reported
    # beside it: that one also carries the launch and the cold prologue.
    flush = algo_bytes < 4 * 126e6
    reps = None
    if flush:
        from paper_2203_05096_b200 import _native as nat

        # x is prefetched into L2 with evict_last and y is written through
        # L2, so the replicas' x + y (not only the whole working set) must
        # exceed 4 x L2 for every step to read its x from HBM
        xy_bytes = 2 * n * vbytes
        n_rep = min(64, max(-(-int(4 * 126e6) // algo_bytes), -(-int(4 * 126e6) // xy_bytes)))
        b = m.base
        dev0 = m.device()
        reps = [(dev0, xd, yd)]
        for _ in range(n_rep - 1):
            d = nat.DeviceMatrix.upload(b.row_ptr, b.col_idx, b.vals, n, n, k=m.k,
                                        sr_ptr=m.group_ptrs[0],
                                        ssr_ptr=m.group_ptrs[1] if m.k == 3 else None)
            reps.append((d, xd.clone(), torch.empty_like(yd)))
        for d, xr, yr in reps:
            ck.spmv_device(d, xr, yr, dims=dims, variant=variant, stream=stream)
        plan_keys = ("tile_cost", "stages", "n_tiles", "gather_first", "ctas_per_sm")
        p0 = {k: dev0.plan()[k] for k in plan_keys}
        assert all({k: d.plan()[k] for k in plan_keys} == p0 for d, _, _ in reps), \
            "replica plans differ"
        scrub = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
        scrub2 = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
        sink = torch.empty((), dtype=torch.float64, device="cuda")
    with ClockSampler(torch.cuda.current_device()) as clk:
        clk.load_until(step, torch.cuda.synchronize)
        torch.cuda.synchronize()
        if flush:
            # one untimed pass over every replica after the clock sampler's
            # load (which ran replica 0 only): the timed steps continue the
            # rotation, each replica last touched len(reps) steps earlier
            for d, xr, yr in reps:
                ck.spmv_device(d, xr, yr, dims=dims, variant=variant, stream=stream)
            ev0.record(stream)
            for i in range(args.steps):
                d, xr, yr = reps[i % len(reps)]
                ck.spmv_device(d, xr, yr, dims=dims, variant=variant, stream=stream)
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / args.steps
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a_ev, b_ev in evs:
                scrub.fill_(1.0)
                sink.copy_(scrub2.sum())
                a_ev.record(stream)
                step()
                b_ev.record(stream)
            torch.cuda.synchronize()
            ms_flushed = sum(a_ev.elapsed_time(b_ev) for a_ev, b_ev in evs) / args.steps
            for _, _, yr in reps[1:]:
                assert torch.equal(yr, yd), "replica outputs differ"
        else:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / args.steps
    gflops = 2.0 * nnz / (ms * 1e-3) / 1e9
    gbs = algo_bytes / (ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # correctness of the timed output against the drop-in host path
    y_dev = yd.double().cpu().numpy()

    # e2e: the public drop-in call with pinned host buffers
    x_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    x_pin[:] = xp
    y_pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    if variant == "strided":
        def host_call():
            ck.spmv_gpu35(m, x_pin, dims, out=y_pin)
        call_text = "paper_2203_05096_b200.spmv_gpu35(m, x_pinned, dims, out=y_pinned)"
    else:
        def host_call():
            ck.spmv_csr3(m, x_pin, out=y_pin)
        call_text = "paper_2203_05096_b200.spmv_csr3(m, x_pinned, out=y_pinned)"
    for _ in range(max(1, args.warmup)):
        host_call()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        host_call()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if not f32:
        assert np.array_equal(y_dev, y_pin), "device-resident and host-path y differ"

    base, y_base = cpu_baseline(m, xp, budget_s=args.cpu_budget)
    # parity of the TIMED output: the device-resident y of the last timed
    # launch against the oracle (the cpu_baseline's own y for the serial
    # order, the strided restatement otherwise)
    want = y_base if variant == "serial" else oracle_y(m, xp, variant, dims.x)
    parity = parity_of(y_dev, want, m, xp, f32)
    if not parity["ok"]:
        raise SystemExit(f"parity check failed: {parity}")
    key = f"{args.config}_{'f32' if f32 else 'f64'}"
    line = {
        "metric": METRIC,
        "value": round(gflops, 2),
        "unit": "GFLOP/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32" if f32 else "f64",
        "data": "synthetic (deterministic grid Laplacian, x ~ U[-1,1) seed 0)",
        "config": {"workload": CONFIG_TEXT.get(args.config, args.config),
                   "config_id": args.config, "n_rows": n, "nnz": nnz,
                   "ssrs_target": params.ssrs, "srs_target": params.srs,
                   "n_sr": m.num_super_rows, "n_ssr": m.num_ssr,
                   "kernel": f"csrk_stream_kernel ({variant})",
                   "plan": {k: v for k, v in m.device().plan(f32=f32).items()
                            if k in ("tile_cost", "stages", "n_tiles", "group_aligned",
                                     "gather_first", "ctas_per_sm", "n_long")},
                   "parallelism": "1 GPU",
                   "l2": ("inputs larger than L2 (algorithmic %.2f GB per step vs 126 MB "
                          "L2); no flush" % (algo_bytes / 1e9)) if not flush else
                         ("inputs larger than L2: the steps rotate through %d resident "
                          "replicas of the matrix, x and y (%.0f MB per step, %.0f MB in "
                          "all, x + y alone %.0f MB), back to back" % (
                              len(reps), algo_bytes / 1e6, len(reps) * algo_bytes / 1e6,
                              len(reps) * 2 * n * vbytes / 1e6))},
        "hbm_gbs": round(gbs, 1),
        **({"single_launch_l2_flushed": {
            "ms": round(ms_flushed, 4),
            "gflops": round(2.0 * nnz / (ms_flushed * 1e-3) / 1e9, 2),
            "frac": round(algo_bytes / (ms_flushed * 1e-3) / 1e9 / measured_peak()[0], 4),
            "how": "each step alone between its own events after a 512 MB write + "
                   "512 MB read L2 flush (includes the launch and the cold prologue)"}}
           if flush else {}),
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(gbs / peak, 4),
                     "peak_source": peak_src,
                     "frac_of_8tbs_nominal": round(gbs / 8000.0, 4),
                     "traffic": ncu_traffic(key),
                     "algorithmic_bytes_per_launch": algo_bytes},
        "e2e": {"value": round(2.0 * nnz / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(x_pin.nbytes),
                "d2h_bytes_per_step": int(y_pin.nbytes),
                "ms_per_step": round(e2e_s * 1e3, 3),
                "call": call_text},
        "cpu_baseline": base,
        "parity": parity,
        "gpu_launches": args.steps * (2 if m.device().plan()["n_long"] > 0 else 1),
        "clocks": clk.summary(),
        "build_seconds": {k: round(v, 2) for k, v in build_t.items()},
    }
    return line


def run_loop(args, log):
    """--config C4 --loop cg|power: BASELINE configs[3], 100 SpMVs as a CG
    inner loop on the 512^3 7-point Laplacian.  The matrix is generated in
    HBM (csrk_stencil) in natural order with uniform 8 / 8 groups (k = 3,
    identity permutation); one step = `--iters` loop iterations captured in
    one CUDA graph."""
    import torch

    from paper_2203_05096_b200 import cg, synthetic
    from paper_2203_05096_b200.bench import spmv_bytes

    torch.cuda.set_device(0)
    side = args.side
    t0 = time.perf_counter()
    dev = synthetic.device_stencil((side, side, side), 7).group_uniform(8, 8)
    t_gen = time.perf_counter() - t0
    n, nnz = dev.n_rows, dev.nnz
    f32 = args.fp32
    dtype = torch.float32 if f32 else torch.float64
    vb = 4 if f32 else 8
    if f32:
        dev.ensure_f32()
    log(f"[bench] C4 loop={args.loop}: n={n} nnz={nnz} generated in HBM in {t_gen:.1f}s")
    g = torch.Generator(device="cuda").manual_seed(0)
    b = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1).to(dtype)
    x = torch.zeros_like(b)
    scratch = tuple(torch.empty_like(b) for _ in range(3))
    iters = args.iters

    def loop(stream):
        if args.loop == "cg":
            x.zero_()
            cg.cg(dev, b, x, iters=iters, stream=stream, scratch=scratch, sync=False)
        else:
            x.copy_(b)
            cg.power_iterations(dev, x, iters=iters, y=scratch[0], stream=stream)

    graph = cg.GraphedLoop(loop)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        clk.load_until(graph.replay, torch.cuda.synchronize, max_s=6.0)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            graph.replay()
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    spmv_flops = 2.0 * nnz * iters
    gflops = spmv_flops / (ms * 1e-3) / 1e9
    # algorithmic bytes per iteration: the SpMV plus the vector work (CG:
    # update reads 4n writes 2n, direction reads 2n writes n, and p.Ap needs
    # no vector traffic of its own when fused into the SpMV's epilogue --
    # power: 2n + 2n).  The count stays 9n whether or not this launch fuses
    # p.Ap (fp64 does; fp32 runs the separate dot kernel, which re-reads p and
    # Ap but is faster overall, csrc/spmv.cu launch_spmv_dot): the roofline is
    # against the algorithm's bytes, not the implementation's.
    fused_dot = (args.loop == "cg" and os.environ.get("CSRK_NO_FUSED_DOT") is None
                 and (not f32 or os.environ.get("CSRK_FUSED_DOT_F32") == "1"))
    vec_words = 9 * n if args.loop == "cg" else 4 * n
    it_bytes = spmv_bytes(n, n, nnz, vb) + vec_words * vb
    gbs = it_bytes * iters / (ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    # e2e through the public API: b from pinned host, x back to pinned host
    b_pin = torch.empty(n, dtype=dtype, pin_memory=True)
    b_pin.copy_(b)
    x_pin = torch.empty(n, dtype=dtype, pin_memory=True)
    e2e_t = []
    for _ in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        bd = b_pin.to("cuda", non_blocking=True)
        xd = torch.zeros_like(bd)
        if args.loop == "cg":
            cg.cg(dev, bd, xd, iters=iters, scratch=scratch, sync=False)
        else:
            xd.copy_(bd)
            cg.power_iterations(dev, xd, iters=iters, y=scratch[0])
        x_pin.copy_(xd, non_blocking=True)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t1)
    e2e_s = sum(e2e_t[1:]) / max(1, len(e2e_t) - 1)
    return {
        "metric": METRIC, "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if f32 else "f64",
        "data": "synthetic (512^3 7-point Laplacian generated in HBM, b ~ U[-1,1))",
        "config": {"workload": f"C4: {iters} SpMVs as a {args.loop} inner loop on the "
                               f"{side}^3 7-point Laplacian, CUDA graph",
                   "config_id": "C4", "n_rows": n, "nnz": nnz, "iterations_per_step": iters,
                   "grouping": "natural order, uniform SR 8 / SSR 8 (identity permutation)",
                   "ms_per_iteration": round(ms / iters, 5),
                   "l2": "inputs larger than L2; no flush", "parallelism": "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(gbs / peak, 4), "peak_source": peak_src,
                     "traffic": None,
                     "algorithmic_bytes_per_iteration": int(it_bytes)},
        "e2e": {"value": round(spmv_flops / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": n * vb, "d2h_bytes_per_step": n * vb,
                "ms_per_step": round(e2e_s * 1e3, 3),
                "call": f"paper_2203_05096_b200.cg.{'cg' if args.loop == 'cg' else 'power_iterations'}"},
        "gpu_launches": args.steps * iters * ((4 if fused_dot else 5) if args.loop == "cg" else 3),
        "clocks": clk.summary(),
    }


REF_DIR = os.path.join(REPO, "baseline", "_ref")
REF_CACHE = os.path.join(REPO, "baseline", "_cache")
B200_PROFILE = os.path.join(REPO, "paper_2203_05096_b200", "data", "b200.json")


def _import_reference():
    """The UNMODIFIED reference package installed at baseline/_ref (pip
    --target of /root/reference/pkg).  The repo root leaves sys.path first so
    its `csrk` alias of this package cannot shadow it; nothing of this repo's
    package (and none of its .so files) is imported on this arm."""
    if not os.path.isfile(os.path.join(REF_DIR, "csrk", "__init__.py")):
        return None
    sys.path[:] = [REF_DIR] + [p for p in sys.path
                               if os.path.abspath(p or os.getcwd()) != REPO]
    for k in [k for k in sys.modules if k == "csrk" or k.startswith("csrk.")]:
        del sys.modules[k]
    import csrk
    if not os.path.abspath(csrk.__file__).startswith(REF_DIR):
        raise RuntimeError(f"reference import resolved to {csrk.__file__}")
    return csrk


def _load_synthetic():
    """The numpy-only input generator (paper_2203_05096_b200/synthetic.py),
    loaded by file path so the package (and its CUDA library) stays out of
    this process -- the same generator the golden script feeds the reference."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_csrk_synthetic", os.path.join(REPO, "paper_2203_05096_b200", "synthetic.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def reference_matrix(ref, cfg: str, log):
    """The config's CSR-k built entirely by the reference: CsrMatrix /
    csr_from_arrays, compute_stats, tune_gpu with the B200 profile JSON (the
    reference's own plugin mechanism, tuning.py:518), band_k, pack_csrk,
    permute_vector.  band_k takes minutes at C2 / C3 / C5 in pure Python, so
    its result (perm.fwd and the level sizes, written by this same code on a
    previous run) is reused from baseline/_cache when the input digest
    matches."""
    import hashlib

    syn = _load_synthetic()
    t0 = time.perf_counter()
    kind, shape, points = syn.CONFIGS[cfg]
    if kind == "stencil":
        n, rp, ci, va = syn.stencil_arrays(shape, points)
        a = ref.CsrMatrix(n, n, rp, ci, va)
    else:
        rows, cols, vals = syn.irregular_triplets(shape)
        a = ref.csr_from_arrays(shape, shape, rows, cols, vals)
        n = a.n_rows
    t_gen = time.perf_counter() - t0
    stats = ref.compute_stats(a)
    params = ref.tune_gpu(stats, ref.load_profile(B200_PROFILE))
    targets = [params.srs, params.ssrs]
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(np.ascontiguousarray(arr).tobytes())
    tag = h.hexdigest()[:16]
    path = os.path.join(REF_CACHE, f"{cfg}_k3_{targets[0]}_{targets[1]}_{tag}.npz")
    t0 = time.perf_counter()
    cached = os.path.exists(path)
    if cached:
        z = np.load(path)
        perm = ref.Permutation.from_forward(z["fwd"].astype(np.int64))
        groups = [z["sizes0"].tolist(), z["sizes1"].tolist()]
    else:
        res = ref.band_k(a, 3, targets)
        perm, groups = res.perm, [list(g) for g in res.level_group_sizes]
        try:
            os.makedirs(REF_CACHE, exist_ok=True)
            np.savez_compressed(path, fwd=np.asarray(perm.fwd, dtype=np.uint32),
                                sizes0=np.asarray(groups[0], dtype=np.int64),
                                sizes1=np.asarray(groups[1], dtype=np.int64))
        except OSError:
            pass
    t_band = time.perf_counter() - t0
    t0 = time.perf_counter()
    m = ref.pack_csrk(a, perm, groups)
    t_pack = time.perf_counter() - t0
    x = np.random.default_rng(0).uniform(-1.0, 1.0, n)
    xp = ref.permute_vector(perm, x)
    log(f"[reference] {cfg}: n={n} nnz={a.nnz} targets {targets} gen {t_gen:.1f}s "
        f"band_k {t_band:.1f}s ({'cached perm' if cached else 'computed'}) pack {t_pack:.1f}s")
    return a, m, x, xp, params, {"gen_s": round(t_gen, 2), "band_k_s": round(t_band, 2),
                                 "band_k_cached": cached, "pack_s": round(t_pack, 2)}


def run_reference(args, log):
    """--impl reference: the reference's own CPU CSR-3 SpMV,
    ``spmv_csr3(m, xp, workers=os.cpu_count())`` (kernels.py:209-221), from
    the unmodified package at baseline/_ref, on the same config, metric and
    (B200-profile) group sizes as this repo's arm.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    ref = _import_reference()
    if ref is None:
        return {"impl": "reference",
                "unavailable": "baseline/_ref/csrk is not installed (pip --target of "
                               "/root/reference/pkg)"}
    if args.config == "C4":
        return {"impl": "reference",
                "unavailable": "C4 (938 M nonzeros): the reference's csr_from_arrays / "
                               "band_k cannot build it in host RAM and time (SURVEY.md 8(d))"}
    a, m, x, xp, params, build_t = reference_matrix(ref, args.config, log)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        ref.spmv_csr3(m, xp, workers=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.spmv_csr3(m, xp, workers=threads)
        times.append(time.perf_counter() - t0)
    mean = sum(times) / len(times)
    val = round(2.0 * a.nnz / mean / 1e9, 4)
    extra = {}
    if args.config == "C1":
        # BASELINE.json names C1 the "reference CPU path": the sequential
        # oracle spmv_csr_ref (kernels.py:97-114), one core, one call
        t0 = time.perf_counter()
        ref.spmv_csr_ref(a, x)
        t_ref = time.perf_counter() - t0
        extra["spmv_csr_ref"] = {"value": round(2.0 * a.nnz / t_ref / 1e9, 4),
                                 "unit": "GFLOP/s", "cores": 1, "seconds": round(t_ref, 3)}
    try:
        cpu_model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                          if ln.startswith("model name")), None)
    except OSError:
        cpu_model = None
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": val,
        "unit": "GFLOP/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(mean * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (deterministic grid Laplacian / irregular rows, x ~ U[-1,1) seed 0)",
        "config": {"workload": CONFIG_TEXT.get(args.config, args.config),
                   "config_id": args.config, "n_rows": a.n_rows, "nnz": a.nnz,
                   "ssrs_target": params.ssrs, "srs_target": params.srs,
                   "n_sr": m.num_super_rows, "n_ssr": m.num_ssr},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads,
                         "kind": "reference", "cpu_model": cpu_model,
                         "sample": f"{args.steps} whole-matrix calls of the unmodified "
                                   "reference csrk.spmv_csr3(m, xp, workers=os.cpu_count()) "
                                   "(kernels.py:209-221, baseline/_ref) on the CSR-k matrix "
                                   "the reference's own band_k + pack_csrk built"},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_seconds": build_t,
        **extra,
    }


def _relaunch_torchrun(n: int, argv) -> None:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *argv]
    print(f"[bench] --gpus {n}: " + " ".join(cmd), file=sys.stderr, flush=True)
    rc = subprocess.run(cmd).returncode
    if rc:
        raise SystemExit(rc)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C2", choices=("C1", "C2", "C3", "C4", "C5"))
    ap.add_argument("--loop", choices=("cg", "power"), default="cg",
                    help="C4 only: the iterative loop around the SpMV")
    ap.add_argument("--iters", type=int, default=100, help="C4: loop iterations per step")
    ap.add_argument("--side", type=int, default=512, help="C4: grid side")
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--exchange", choices=("halo", "allgather"), default=None,
                    help="N > 1: x exchange (default halo; allgather = the literal "
                         "north-star collective)")
    ap.add_argument("--partition", choices=("blocks", "slab"), default="blocks",
                    help="N > 1, C2: SSR row blocks of the CSR-k matrix (strong scaling, "
                         "default) or round 1's weak-scaling z-slabs")
    ap.add_argument("--mg", choices=("torch", "native"), default="native",
                    help="N > 1, SSR blocks: exchange through torch.distributed (DistSpMV) "
                         "or the library's C-ABI (csrk_mg_*, NativeDistSpMV)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="N > 1 with --mg native: time eager steps instead of one CUDA "
                         "graph of the K steps")
    ap.add_argument("--probe-launch", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None and args.impl == "ours":
        # one process per GPU: re-launch this command under torchrun
        return _relaunch_torchrun(args.gpus, sys.argv[1:] if argv is None else argv)
    if world_env is not None and args.impl == "ours" and int(world_env) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))

    def log(msg):
        if rank == 0:
            print(msg, file=sys.stderr, flush=True)

    # libraries may write to the process's stdout (NCCL prints its version
    # line at communicator creation): keep fd 1 for the one JSON line
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        line = _run(args, log)
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


def _run(args, log):
    if args.probe_launch:  # tests: the process layout only, no GPU work
        return {"probe": True, "world_size": int(os.environ.get("WORLD_SIZE", "1")),
                "n_gpus": args.gpus, "torchrun": "LOCAL_RANK" in os.environ}
    if args.impl == "reference":
        line = run_reference(args, log)
    elif args.config == "C4" and int(os.environ.get("WORLD_SIZE", "1")) == 1 and \
            os.environ.get("CSRK_DIST") != "1":
        line = run_loop(args, log)
    else:
        line = run_ours(args, log)
    return line


if __name__ == "__main__":
    main()
