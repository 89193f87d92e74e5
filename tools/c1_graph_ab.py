"""Small configs: are back-to-back rotated steps bound by the host's launch
rate?  Times the bench's replica rotation (see bench.py run_ours) eagerly
and as one CUDA graph of the same K launches (programmatic-dependent-launch
edges captured), interleaved, and the host time to enqueue one eager step.

    python tools/c1_graph_ab.py [C1] [--fp32] [steps] [rounds]
"""
from __future__ import annotations

import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import _native as nat  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    f32 = "--fp32" in sys.argv
    cfg = args[0] if args else "C1"
    steps = int(args[1]) if len(args) > 1 else 64
    rounds = int(args[2]) if len(args) > 2 else 5
    torch.cuda.set_device(0)
    a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
    n, nnz = a.n_rows, a.nnz
    dims = params.block_dims
    variant = "strided" if params.kernel_variant.value == "cuda35" else "serial"
    dt = torch.float32 if f32 else torch.float64
    vb = 4 if f32 else 8
    algo = spmv_bytes(n, n, nnz, vb)
    n_rep = min(64, max(-(-int(4 * 126e6) // algo), -(-int(4 * 126e6) // (2 * n * vb))))
    b = m.base
    xd = torch.from_numpy(xp).to("cuda", dt)
    reps = [(m.device(), xd, torch.empty(n, dtype=dt, device="cuda"))]
    for _ in range(n_rep - 1):
        d = nat.DeviceMatrix.upload(b.row_ptr, b.col_idx, b.vals, n, n, k=m.k,
                                    sr_ptr=m.group_ptrs[0],
                                    ssr_ptr=m.group_ptrs[1] if m.k == 3 else None)
        reps.append((d, xd.clone(), torch.empty(n, dtype=dt, device="cuda")))

    def run(stream):
        for i in range(steps):
            d, xr, yr = reps[(i + 1) % n_rep]
            ck.spmv_device(d, xr, yr, dims=dims, variant=variant, stream=stream)

    stream = torch.cuda.current_stream()
    run(stream)
    torch.cuda.synchronize()
    from paper_2203_05096_b200.cg import GraphedLoop
    g = GraphedLoop(run)
    peak, _ = bench.measured_peak()
    res = {"eager": [], "graph": [], "host_enqueue_us": []}
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        t0 = time.perf_counter()
        run(stream)
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        res["eager"].append(e0.elapsed_time(e1) / steps)
        res["host_enqueue_us"].append((t1 - t0) / steps * 1e6)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        res["graph"].append(e0.elapsed_time(e1) / steps)
    for k in ("eager", "graph"):
        ms = sorted(res[k])[len(res[k]) // 2]
        print(json.dumps({"config": cfg, "f32": f32, "mode": k, "replicas": n_rep, "steps": steps,
                          "ms_median": round(ms, 5), "all": [round(v, 5) for v in res[k]],
                          "frac": round(algo / (ms * 1e-3) / 1e9 / peak, 4)}))
    print(json.dumps({"config": cfg, "f32": f32, "host_enqueue_us_per_step":
                      [round(v, 1) for v in res["host_enqueue_us"]]}))


if __name__ == "__main__":
    main()
