import sys; sys.path.insert(0,'.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]); method = sys.argv[2]; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = CONFIGS[cfg]
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
for _ in range(reps):
    r = api.decompose_device(a.data_ptr(), c["dims"], method, "l2r" if method == "ulv" else "r2l", a_is_device_ptr=True, **kw)
    print(r.report().ranks_chosen, [(x["m"], x["n"], x["steps"]) for x in r.report().cuts], flush=True)
