"""Time the pinned host pipeline (spmv_csr3 with pinned x / y) for several
chunk shapes (CSRK_PIPE_SHAPE, csrc/abi.cu pipe_weights):
    python tools/pipe_shapes.py C2 u16 r12 r8 ..."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402

cfg = sys.argv[1]
a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
n = a.n_rows
xn = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
yn = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
xn[:] = xp
strided = params.kernel_variant.value == "cuda35"


def call():
    if strided:
        ck.spmv_gpu35(m, xn, params.block_dims, out=yn)
    else:
        ck.spmv_csr3(m, xn, out=yn)


ref = None
for spec in sys.argv[2:]:
    shape, d2h, xcut = (spec.split(":") + ["", ""])[:3]
    os.environ["CSRK_PIPE_SHAPE"] = shape
    os.environ["CSRK_PIPE_D2H"] = d2h or "host"
    os.environ["CSRK_PIPE_XCUT"] = xcut or "footprint"
    for _ in range(3):
        call()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    if ref is None:
        ref = yn.copy()
    assert np.array_equal(ref, yn)
    print(f"{cfg} shape {spec:12s} mean {np.mean(ts) * 1e3:.3f} ms  median "
          f"{np.median(ts) * 1e3:.3f} ms  min {np.min(ts) * 1e3:.3f} ms", flush=True)
os.environ["CSRK_PIPE_TRACE"] = "1"
for spec in sys.argv[-2:]:
    shape, d2h, xcut = (spec.split(":") + ["", ""])[:3]
    os.environ["CSRK_PIPE_SHAPE"] = shape
    os.environ["CSRK_PIPE_D2H"] = d2h or "host"
    os.environ["CSRK_PIPE_XCUT"] = xcut or "footprint"
    call()
