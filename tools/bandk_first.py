"""First-call cost of the device Band-k as the full-size test sees it:
a.device() upload, then band_k twice, phases on stderr (CSRK_BANDK_PROFILE)."""
import os
import sys
import time

os.environ["CSRK_BANDK_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
targets = {"C2": [7, 6], "C3": [10, 20], "C5": [14, 9]}[cfg]
t = time.perf_counter()
n, rp, ci, va = synthetic.config_arrays(cfg)
a = ck.CsrMatrix(n, n, rp, ci, va)
print(cfg, f"arrays {time.perf_counter() - t:.2f}s", file=sys.stderr, flush=True)
t = time.perf_counter()
a.device()
print(cfg, f"a.device() {time.perf_counter() - t:.2f}s", file=sys.stderr, flush=True)
for i in range(2):
    t = time.perf_counter()
    ck.band_k(a, 3, targets, backend="device")
    print(cfg, f"band_k call {i} {time.perf_counter() - t:.2f}s", file=sys.stderr, flush=True)
