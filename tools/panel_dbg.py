import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2203_05096_b200 as ck
from paper_2203_05096_b200 import synthetic
from oracle import oracle as O
r, c, v = synthetic.irregular_triplets(120000, seed=5)
a = ck.csr_from_arrays(120000, 120000, r, c, v)
res = ck.band_k(a, 3, [7, 11])
m = ck.pack_csrk(a, res.perm, res.level_group_sizes)
b = m.base
x = np.random.default_rng(0).uniform(-1.0, 1.0, b.n_rows)
dev = m.device()
dev.set_layout(1)
y = ck.spmv_csr3(m, x)
want = O.spmv_serial(b.row_ptr, b.col_idx, b.vals, x)
bad = np.flatnonzero(y != want)
print("plan", dev.plan())
print("bad", len(bad), bad[:20])
rp = b.row_ptr.astype(np.int64)
print("bad row lens", np.diff(rp)[bad[:20]])
