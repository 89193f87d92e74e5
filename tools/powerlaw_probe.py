"""Power-law row lengths (the paper's failure mode): the
serial order against the strided order with 4..32 lanes, f64, one B200.
    python tools/powerlaw_probe.py [n_rows] [max_len]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200.bench import spmv_bytes  # noqa: E402


def powerlaw_triplets(n, max_len, seed=0, alpha=2.0):
    rng = np.random.default_rng(seed)
    lens = np.minimum(max_len, np.floor(rng.pareto(alpha - 1.0, n) * 3 + 1)).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    cols = rng.integers(0, n, len(rows))
    starts = np.zeros(n, dtype=np.int64)
    np.cumsum(lens[:-1], out=starts[1:])
    cols[starts] = np.arange(n)
    return rows, cols, rng.uniform(0.5, 1.5, len(rows))


def med(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def build_powerlaw(n, max_len):
    """(csr, csrk matrix, stats, tuned params) of one power-law case."""
    r, c, v = powerlaw_triplets(n, max_len)
    a = ck.csr_from_arrays(n, n, r, c, v)
    st = ck.compute_stats(a)
    p = ck.tune_gpu(st, ck.b200_profile())
    res = ck.band_k(a, 3, [p.srs, p.ssrs])
    return a, ck.pack_csrk(a, res.perm, res.level_group_sizes), st, p


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    for max_len in [int(v) for v in (sys.argv[2:] or ["1000", "20000"])]:
        a, m, st, p = build_powerlaw(n, max_len)
        x = torch.rand(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        byts = spmv_bytes(n, n, a.nnz, 8)
        print(f"max_len {max_len}: nnz {a.nnz} rd {st.rdensity:.2f} var {st.variance:.1f} "
              f"max_row {st.max_row_nnz} tuned {p.kernel_variant.value} {p.block_dims}", flush=True)
        for variant, nx in [("serial", 0), ("strided", 4), ("strided", 8), ("strided", 16),
                            ("strided", 32)]:
            dims = ck.BlockDims(max(nx, 1), 1, 1)
            ms = med(lambda: ck.spmv_device(m, x, y, dims=dims, variant=variant))
            print(f"  {variant:8s} nx {nx:2d}: {ms * 1e3:8.1f} us  {byts / ms / 1e6:6.0f} GB/s",
                  flush=True)


if __name__ == "__main__":
    main()
