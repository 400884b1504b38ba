"""Wall vs device time per decomposition (diagnostics for host-side stalls)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200._native import lib
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
c = CONFIGS[cfg]
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
lib().ttg_synchronize()
if len(sys.argv) > 2 and sys.argv[2] == "prof":
    lib().ttg_profile_enable(1)
s = torch.cuda.ExternalStream(lib().ttg_stream())
for it in range(8):
    for m, sw in (("ulv", "l2r"), ("urv", "r2l")):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        lib().ttg_synchronize()
        f0 = torch.cuda.memory.mem_get_info()[0]
        t1 = time.perf_counter(); e0.record(s)
        r = api.decompose_device(a.data_ptr(), c["dims"], m, sw, a_is_device_ptr=True, **kw)
        e1.record(s); t2 = time.perf_counter(); e1.synchronize(); t3 = time.perf_counter()
        f1 = torch.cuda.memory.mem_get_info()[0]
        print(f"{m} host {1e3*(t2-t1):7.1f} ms  +tail {1e3*(t3-t2):6.1f}  dev {e0.elapsed_time(e1):7.1f} ms  free {f0/2**30:.1f}->{f1/2**30:.1f} GiB", flush=True)
        del r
