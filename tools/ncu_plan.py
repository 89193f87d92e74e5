"""Run the streaming kernel of one config under a given plan / gather mode
(for ncu captures of plan variants):
    python tools/ncu_plan.py C5 TILE_COST STAGES GATHER [serial|strided] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_05096_b200 as ck  # noqa: E402

cfg, tc, st, g = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
CTAS = int(os.environ.get("CTAS", "0"))
a, m, xp, params, _ = bench.build_matrix(cfg, lambda s: print(s, file=sys.stderr))
variant = sys.argv[5] if len(sys.argv) > 5 else (
    "strided" if params.kernel_variant.value == "cuda35" else "serial")
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
dev = m.device()
dev.set_plan(tc, 0, st)
dev.set_schedule(g, CTAS)
dev.set_cut_mode(int(os.environ.get("CUT", "0")))
xd = torch.from_numpy(xp).cuda()
yd = torch.empty_like(xd)
for _ in range(reps):
    ck.spmv_device(m, xd, yd, dims=params.block_dims, variant=variant)
torch.cuda.synchronize()
print("plan", dev.plan(), variant)
