import sys, time, ctypes, subprocess
sys.path.insert(0, '.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200._native import lib
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prof = len(sys.argv) > 2 and sys.argv[2] == "prof"
smi = len(sys.argv) > 3 and sys.argv[3] == "smi"
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
c = CONFIGS[cfg]
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
lib().ttg_profile_enable(1 if prof else 0)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"], stdout=subprocess.DEVNULL) if smi else None
for it in range(8):
    t0 = time.perf_counter()
    for m, s in (("ulv", "l2r"), ("urv", "r2l")):
        t1 = time.perf_counter()
        r = api.decompose_device(a.data_ptr(), c["dims"], m, s, a_is_device_ptr=True, **kw)
        t2 = time.perf_counter()
        print(f"  {m} {1e3*(t2-t1):.1f} ms", end="")
        del r
    print(f" | step {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
if p: p.terminate()
