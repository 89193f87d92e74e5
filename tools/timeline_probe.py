"""Per-CTA timeline of one streaming-kernel launch (diagnostic build).

    bash tools/build_variant.sh tl -DCSRK_TIMELINE=1
    CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_tl.so python tools/timeline_probe.py C1

Runs the config's SpMV after a 512 MB write + read L2 flush, then reads the
per-CTA slots the kernel wrote (csrk_debug_timeline): entry %globaltimer
(aligns the SMs), and SM-clock cycles after entry of the producer's first TMA
issue, the consumers' first full stage, their last stage released, the
producer's exit, and the tile count.  Prints the spread of each event across
CTAs in microseconds from the first CTA's entry, and the kernel's event time.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import _native  # noqa: E402


def pct(a, q):
    return round(float(np.percentile(a, q)), 2)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
    n = a.n_rows
    dims = params.block_dims
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    xd = torch.from_numpy(xp).to("cuda", torch.float64)
    yd = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    scrub = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    scrub2 = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")
    lib = _native.lib()
    fn = lib.csrk_debug_timeline
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    fn.restype = C.c_int
    sm_hz = torch.cuda.get_device_properties(0).clock_rate * 1e3 if hasattr(
        torch.cuda.get_device_properties(0), "clock_rate") else None
    for _ in range(3):
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant, stream=stream)
    torch.cuda.synchronize()
    for rep in range(reps):
        scrub.fill_(1.0)
        sink.copy_(scrub2.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ncta = 4096
        buf = (C.c_ulonglong * (ncta * 6))()
        assert fn(buf, ncta) == 0
        t = np.frombuffer(buf, dtype=np.uint64).reshape(ncta, 6).astype(np.float64)
        used = t[:, 0] > 0
        t = t[used]
        # one launch only: CTAs of this launch have entries within ~50 us
        g0 = t[:, 0].min()
        t = t[t[:, 0] - g0 < 1e5]
        ent = (t[:, 0] - g0) / 1e3  # us
        # SM clock under load for cycle -> us (nvidia-smi's SM clock is what the
        # clock64 counter ticks at); fall back to the device's max clock
        clk = float(os.environ.get("TL_SM_MHZ", "0")) or (sm_hz / 1e6 if sm_hz else 1965.0)
        cyc = lambda c: c / clk  # cycles -> us at clk MHz
        first_issue = ent + cyc(t[:, 1])
        first_full = ent + cyc(t[:, 2])
        cons_exit = ent + cyc(t[:, 3])
        prod_exit = ent + cyc(t[:, 4])
        tiles = t[:, 5]
        rec = {
            "config": cfg, "rep": rep, "event_ms": round(e0.elapsed_time(e1), 5),
            "ctas": int(len(t)), "sm_mhz_assumed": clk,
            "entry_us": [pct(ent, 0), pct(ent, 50), pct(ent, 100)],
            "first_tma_issue_us": [pct(first_issue, 0), pct(first_issue, 50), pct(first_issue, 100)],
            "first_full_us": [pct(first_full, 0), pct(first_full, 50), pct(first_full, 100)],
            "producer_exit_us": [pct(prod_exit, 0), pct(prod_exit, 50), pct(prod_exit, 100)],
            "consumer_exit_us": [pct(cons_exit, 0), pct(cons_exit, 10), pct(cons_exit, 50),
                                 pct(cons_exit, 90), pct(cons_exit, 100)],
            "tiles_per_cta": [int(tiles.min()), int(tiles.max())],
        }
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
