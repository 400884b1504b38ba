"""cfg5 through the sharded engine at NCCL world size 1 (diagnostics: per-cut timing)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = CONFIGS[cfg]
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
comm = api.loopback_group(1)[0] if (len(sys.argv) > 2 and sys.argv[2] == "loop") else api.nccl_comm(api.nccl_unique_id(), 1, 0)
if "reserve" in sys.argv:
    from paper_2501_07904_b200._native import lib
    print("reserve", lib().ttg_reserve(24 << 30))
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
for it in range(6):
    t0 = time.perf_counter()
    r = api.decompose_sharded(a.data_ptr(), c["dims"], comm, "urv", "r2l", a_is_device_ptr=True, **kw)
    print(f"sharded {1e3*(time.perf_counter()-t0):.1f} ms", r.report().ranks_chosen, flush=True)
    t0 = time.perf_counter()
    r = api.decompose_device(a.data_ptr(), c["dims"], "urv", "r2l", a_is_device_ptr=True, **kw)
    print(f"single  {1e3*(time.perf_counter()-t0):.1f} ms", r.report().ranks_chosen, flush=True)
