"""Device Band-k + pack + SpMV on a small stencil and an irregular matrix (sanitizer target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_05096_b200 as ck  # noqa: E402
from paper_2203_05096_b200 import synthetic  # noqa: E402

n, rp, ci, va = synthetic.stencil_arrays((20, 22, 24), 7, values="uniform")
a = ck.CsrMatrix(n, n, rp, ci, va)
r1 = ck.band_k(a, 3, [6, 7], backend="device")
r2 = ck.band_k(a, 3, [6, 7], backend="host")
assert np.array_equal(r1.perm.fwd, r2.perm.fwd)
rows, cols, vals = synthetic.irregular_triplets(30000, max_len=19, reach=2000)
b = ck.csr_from_arrays(30000, 30000, rows, cols, vals)
r3 = ck.band_k(b, 3, [14, 9], backend="device")
r4 = ck.band_k(b, 3, [14, 9], backend="host")
assert np.array_equal(r3.perm.fwd, r4.perm.fwd)
m = ck.pack_csrk(b, r3.perm, r3.level_group_sizes)
x = np.random.default_rng(0).uniform(-1, 1, 30000)
ck.spmv_csr3(m, x)
print("bandk sanitizer target ok")
