import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2501_07904_b200 import api
from tests.fixtures import shifted_hilbert
dims = [10]*4
a = shifted_hilbert(dims)
for method in ["urv", "ulv"]:
    res = api.decompose_device(a, dims, method, "r2l" if method == "urv" else "l2r", eps=1e-6)
    rep = res.report()
    print(method, rep.ranks_chosen, [ (c["steps"], c["p"], c["extensions"]) for c in rep.cuts], flush=True)
