"""python scripts/dump_cores.py CFG OUT.npz: ULV + URV cores of a BASELINE config (bitwise
comparisons between engine variants selected by environment switches; diagnostics)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]); out = sys.argv[2]
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
c = CONFIGS[cfg]
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
arrs = {}
for m, s in (("ulv", "l2r"), ("urv", "r2l")):
    r = api.decompose_device(a.data_ptr(), c["dims"], m, s, a_is_device_ptr=True, **kw)
    for i in range(r.order()):
        arrs[f"{m}_{i}"] = r.core(i)
    print(m, r.report().ranks_chosen, flush=True)
np.savez(out, **arrs)
