import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2501_07904_b200 import api
rng = np.random.default_rng(0)
cores = [rng.standard_normal((1,5,3)), rng.standard_normal((3,4,2)), rng.standard_normal((2,6,1))]
x = api.reconstruct(cores)
# numpy contraction
t = np.einsum('aib,bjc,ckd->ijk', *cores)
print("recon err", np.max(np.abs(x - t)), np.max(np.abs(t)))
for (m,n,k) in [(5,6,3),(64,64,16),(70,33,17),(200,100,5)]:
    cores = [rng.standard_normal((1,m,k)), rng.standard_normal((k,n,1))]
    x = api.reconstruct(cores)
    t = cores[0][0] @ cores[1][:,:,0]
    print(m,n,k, np.max(np.abs(x - t)))
