import sys, time; sys.path.insert(0,'.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, bernoulli_mask, CONFIGS
c = CONFIGS[4]
dev = torch.device("cuda", 0)
m = build(4, dev); mask = bernoulli_mask(m.numel(), dev)
obs = (m * mask).contiguous(); y = obs.clone()
torch.cuda.synchronize()
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tr = api.complete_tol(y.data_ptr(), obs.data_ptr(), mask.data_ptr(), c["dims"], c["eps"], iters, truth_ptr=m.data_ptr())
for i in range(iters):
    print(i, tr.ranks[i][5:8], "rse_obs %.3e rse_full %.6f psnr %.3f t %.0f ms" % (tr.rse_observed[i], tr.rse_full[i], tr.psnr[i], tr.wall_time_ms[i]))
