"""Sequential vs concurrent (two host threads, one stream each) ULV + URV decompositions of
a BASELINE config through the public API from pinned host memory (experiment)."""
import sys, time, threading
sys.path.insert(0, '.')
import torch
from paper_2501_07904_b200 import api
from paper_2501_07904_b200.inputs import build, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = CONFIGS[cfg]
a = build(cfg, torch.device("cuda", 0)); torch.cuda.synchronize()
host = torch.empty(a.numel(), dtype=torch.float64, pin_memory=True); host.copy_(a.reshape(-1)); torch.cuda.synchronize()
kw = dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])
runs = (("ulv", "l2r"), ("urv", "r2l"))
out = {}
def one(m, s, ptr, dev):
    r = api.decompose_device(ptr, c["dims"], m, s, a_is_device_ptr=dev, **kw)
    out[m] = r.report().ranks_chosen
    del r
for mode, ptr, dev in (("host", host.data_ptr(), False), ("device", a.data_ptr(), True)):
    for conc in (False, True):
        ts = []
        for it in range(reps):
            t0 = time.perf_counter()
            if conc:
                th = [threading.Thread(target=one, args=(m, s, ptr, dev)) for m, s in runs]
                for x in th: x.start()
                for x in th: x.join()
            else:
                for m, s in runs: one(m, s, ptr, dev)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{mode} {'concurrent' if conc else 'sequential'}: " + " ".join(f"{x:.1f}" for x in ts) + f" ms  ranks {out}", flush=True)

# independent worker threads: each thread runs all `reps` decompositions of its kind
def loop(m, s, ptr, dev, n):
    for _ in range(n):
        one(m, s, ptr, dev)
for mode, ptr, dev in (("host", host.data_ptr(), False),):
    t0 = time.perf_counter()
    th = [threading.Thread(target=loop, args=(m, s, ptr, dev, reps)) for m, s in runs]
    for x in th: x.start()
    for x in th: x.join()
    print(f"{mode} independent threads: {1e3 * (time.perf_counter() - t0) / reps:.1f} ms per step", flush=True)
