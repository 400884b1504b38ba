import sys, time; sys.path.insert(0,'.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, bernoulli_mask, CONFIGS
c = CONFIGS[4]
dev = torch.device("cuda", 0)
m = build(4, dev); mask = bernoulli_mask(m.numel(), dev)
y = m * mask
torch.cuda.synchronize()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    r = api.decompose_device(y.data_ptr(), c["dims"], "urv", "r2l", a_is_device_ptr=True, eps=c["eps"])
    rep = r.report()
    t1 = time.perf_counter()
    print(it, rep.ranks_chosen, "%.1f ms" % (1e3*(t1-t0)), [(x["m"], x["n"], x["steps"], x["extensions"]) for x in rep.cuts], flush=True)
    print("rse vs y", r.rse(y.data_ptr(), on_device=True))
