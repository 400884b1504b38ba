"""cudaMallocAsync pool growth cost (diagnostics)."""
import time
from cuda.bindings import runtime as rt, driver as dr
err, dev = rt.cudaGetDevice()
err, pool = rt.cudaDeviceGetDefaultMemPool(0)
thr = dr.cuuint64_t(2**64 - 1)
print(rt.cudaMemPoolSetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold, thr))
err, s = rt.cudaStreamCreateWithFlags(1)
def alloc(n):
    t = time.perf_counter(); e, p = rt.cudaMallocAsync(n, s); rt.cudaStreamSynchronize(s); return p, 1e3*(time.perf_counter()-t)
for it in range(4):
    out = []
    ps = []
    for n in [1 << 30, 1 << 30, 1 << 30, 3 << 28, 5 << 27]:
        p, ms = alloc(n); ps.append(p); out.append(f"{ms:.2f}")
    for p in ps: rt.cudaFreeAsync(p, s)
    rt.cudaStreamSynchronize(s)
    err, used = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    print("iter", it, "alloc ms", out, "reserved GB", int(used) / 2**30, flush=True)
