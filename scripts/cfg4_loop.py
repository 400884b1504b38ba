"""Config 4 (completion) on the device: the 20-iteration rank-adaptive loop through
api.complete (ttg_complete), timed with CUDA events; prints JSON (per-iteration ranks, RSE,
wall ms). Usage: python scripts/cfg4_loop.py [iters]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_07904_b200 import api, inputs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m = inputs.mri_like()
mask = inputs.bernoulli_mask(m.size, seed=41)
lin = np.flatnonzero(mask).astype(np.int64)
dl = torch.from_numpy(lin).cuda()
dv = torch.from_numpy(m[lin]).cuda()
dt = torch.from_numpy(m).cuda()
torch.cuda.synchronize()
# warm-up: one iteration
api.complete(dl.data_ptr(), dv.data_ptr(), [4] * 12, eps=1e-3, retraction="urv", refine_passes=1, max_iters=1,
             stop_tol=0.0, truth=dt.data_ptr(), on_device=True, count=lin.size, dense_cap=20_000_000)
torch.cuda.synchronize()
t0 = time.perf_counter()
c = api.complete(dl.data_ptr(), dv.data_ptr(), [4] * 12, eps=1e-3, retraction="urv", refine_passes=1,
                 max_iters=iters, stop_tol=0.0, truth=dt.data_ptr(), on_device=True, count=lin.size,
                 dense_cap=20_000_000)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tr = c.trace
print(json.dumps({"iterations": iters, "wall_s": wall, "s_per_iteration": wall / (iters + 1),
                  "note": "iterations + the initial guess (iters + 1 retractions)",
                  "ranks_mid": [r[6] for r in tr.ranks], "rse_full": tr.rse_full, "initial": tr.initial,
                  "status": tr.status}))
