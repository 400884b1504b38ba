"""Decompose the same tensor twice and report the first cut whose results differ."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, bernoulli_mask, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
dev = torch.device("cuda", 0)
a = build(cfg, dev)
if cfg == 4:
    a = (a * bernoulli_mask(a.numel(), dev)).contiguous()
torch.cuda.synchronize()
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
method = sys.argv[2] if len(sys.argv) > 2 else "urv"
runs = []
for _ in range(3):
    r = api.decompose_device(a.data_ptr(), c["dims"], method, "l2r" if method == "ulv" else "r2l", a_is_device_ptr=True, **kw)
    rep = r.report()
    runs.append((rep, [r.core(k) for k in range(len(c["dims"]))]))
for i in range(1, len(runs)):
    ra, ca = runs[0]; rb, cb = runs[i]
    print("run", i, "ranks equal", ra.ranks_chosen == rb.ranks_chosen)
    for j, (x, y) in enumerate(zip(ra.cuts, rb.cuts)):
        same = x["steps"] == y["steps"] and len(x["diag"]) == len(y["diag"]) and np.array_equal(x["diag"], y["diag"])
        if not same:
            n = min(len(x["diag"]), len(y["diag"]))
            d = np.flatnonzero(x["diag"][:n] != y["diag"][:n])
            print("  cut", j, "differs: steps", x["steps"], y["steps"], "rank", x["rank"], y["rank"], "first diag diff at", d[:3], x["diag"][d[:1]], y["diag"][d[:1]])
    print("  cores equal:", all(np.array_equal(p, q) for p, q in zip(ca, cb)))
