"""TTG_PHASES=1 python scripts/phases.py CFG [REPS]: per-phase event totals (printed at exit)
of REPS ULV+URV decompositions of a BASELINE config (diagnostics)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
c = CONFIGS[cfg]
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
meths = (("ulv", "l2r"), ("urv", "r2l")) if cfg != 5 else (("urv", "r2l"),)
for it in range(reps):
    t0 = time.perf_counter()
    for m, s in meths:
        r = api.decompose_device(a.data_ptr(), c["dims"], m, s, a_is_device_ptr=True, **kw)
        del r
    print(f"rep {it}: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
