"""Probe managed-memory support on the box: per-allocation and total limits
of cudaMallocManaged (the C5 oversubscription footprint needs > HBM)."""
import ctypes as C, sys, time
rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
for gib in (12, 16, 24, 32, 48):
    p = C.c_void_p()
    e = rt.cudaMallocManaged(C.byref(p), C.c_size_t(gib << 30), 1)
    print(f"cudaMallocManaged({gib} GiB) -> {e}", flush=True)
    if e == 0: rt.cudaFree(p)
    else: rt.cudaGetLastError()
ptrs = []
t0 = time.time()
for i in range(40):
    p = C.c_void_p()
    e = rt.cudaMallocManaged(C.byref(p), C.c_size_t(8 << 30), 1)
    if e != 0:
        print(f"8 GiB chunk #{i} -> {e}"); rt.cudaGetLastError(); break
    ptrs.append(p)
print(f"total managed via 8 GiB chunks: {8*len(ptrs)} GiB in {time.time()-t0:.1f}s", flush=True)
# touch: prefetch a chunk to device and one to host
if ptrs:
    s = rt.cudaMemPrefetchAsync(ptrs[0], C.c_size_t(8 << 30), 0, None); print("prefetch dev", s, rt.cudaDeviceSynchronize())
    s = rt.cudaMemPrefetchAsync(ptrs[-1], C.c_size_t(8 << 30), -1, None); print("prefetch cpu", s, rt.cudaDeviceSynchronize())
for p in ptrs: rt.cudaFree(p)
