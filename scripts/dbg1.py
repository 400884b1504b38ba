import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import ref
from paper_2501_07904_b200 import api
from tests.fixtures import cfg1
from tests.replay import replay
a, dims, ranks = cfg1(ref)
for method in ["urv","ulv"]:
    sweep = "l2r" if method=="ulv" else "r2l"
    res = api.decompose_device(a, dims, method, sweep, ranks=ranks)
    rep = res.report()
    cuts = replay(ref, a, dims, method, ranks=ranks)
    print(method, rep.ranks_chosen, rep.step_errors, res.rse(a))
    for g, r in zip(rep.cuts, cuts):
        print(" gpu", g["m"], g["n"], g["steps"], g["diag"])
        print(" ref", r["m"], r["n"], r["diag"])
    rr = ref.decompose(a, dims, method, sweep, ranks=ranks)
    for k,(c1,c2) in enumerate(zip(res.core(0) if False else [res.core(i) for i in range(4)], rr.cores)):
        print(" core",k,c1.shape,c2.shape, np.max(np.abs(np.abs(c1)-np.abs(c2))))
