"""C1 timing A/B: how the L2 flush between steps shapes the per-step event
time.  A 512 MB write leaves the L2 full of DIRTY scrub lines; the SpMV's
reads then evict them and the write-backs share HBM with the matrix stream.
ncu's --cache-control all instead starts each replay from a clean, invalidated
L2.  Modes (each interleaved, R rounds of S steps):

  write      scrub.fill_ (the bench's round-2 flush)
  write+read scrub.fill_ then a read-only pass over a second 512 MB buffer
             (the L2 ends clean: the dirty scrub lines are written back
             before the timed region)
  none       back-to-back, no flush (L2-warm: NOT a valid C1 number)

    python tools/c1_flush_ab.py [C1] [steps] [rounds]
"""
from __future__ import annotations

import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    torch.cuda.set_device(0)
    a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
    n, nnz = a.n_rows, a.nnz
    dims = params.block_dims
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    xd = torch.from_numpy(xp).to("cuda", torch.float64)
    yd = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    algo = spmv_bytes(n, n, nnz, 8)
    peak, _ = bench.measured_peak()
    scrub = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    scrub2 = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")

    def step():
        ck.spmv_device(m, xd, yd, dims=dims, variant=variant, stream=stream)

    def flush(mode):
        if mode in ("write", "write+read"):
            scrub.fill_(1.0)
        if mode in ("write+read", "read"):
            sink.copy_(scrub2.sum())

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    res = {k: [] for k in ("write", "write+read", "read", "none")}
    for _ in range(rounds):
        for mode in res:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)]
            for e0, e1 in evs:
                flush(mode)
                e0.record(stream)
                step()
                e1.record(stream)
            torch.cuda.synchronize()
            res[mode].append(sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps)
    for mode, v in res.items():
        ms = sorted(v)[len(v) // 2]
        print(json.dumps({"config": cfg, "flush": mode, "ms_median": round(ms, 5),
                          "ms_all": [round(t, 5) for t in v],
                          "gbs": round(algo / (ms * 1e-3) / 1e9, 1),
                          "frac": round(algo / (ms * 1e-3) / 1e9 / peak, 3)}))


if __name__ == "__main__":
    main()
