"""Phase timing of the device Band-k (CSRK_BANDK_PROFILE=1) on a config."""
import os, sys, time
os.environ["CSRK_BANDK_PROFILE"] = "1"
sys.path.insert(0, ".")
import paper_2203_05096_b200 as ck
from paper_2203_05096_b200 import synthetic
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
targets = {"C2": [7, 6], "C3": [10, 20], "C5": [14, 9]}[cfg]
n, rp, ci, va = synthetic.config_arrays(cfg)
a = ck.CsrMatrix(n, n, rp, ci, va, _trusted=True)
a.device()
for backend in ("device", "device"):
    t = time.perf_counter(); ck.band_k(a, 3, targets, backend=backend)
    print(cfg, backend, f"{time.perf_counter() - t:.2f}s", file=sys.stderr, flush=True)
