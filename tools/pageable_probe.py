"""Host-side costs for end-to-end runs from ordinary (pageable) numpy arrays:
cudaHostRegister / Unregister of a large array, multi-threaded memcpy between
pageable and page-locked memory, and the device's pageable-memory-access
attribute.   python tools/pageable_probe.py [--gib 8]"""
import argparse
import ctypes
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=8)
a = ap.parse_args()
n = int(a.gib * (1 << 30) // 8)
cu = torch.cuda.cudart()
print("pageableMemoryAccess:", torch.cuda.get_device_properties(0))
rt = ctypes.CDLL("libcudart.so") if False else None
x = np.empty(n)
t = time.perf_counter(); x.fill(1.0); print(f"first touch {a.gib} GiB: {time.perf_counter()-t:.2f} s")
t = time.perf_counter()
r = cu.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
tr = time.perf_counter() - t
print(f"cudaHostRegister {a.gib} GiB: {tr:.2f} s ({x.nbytes/tr/1e9:.1f} GB/s), rc={r}")
d = torch.empty(n, dtype=torch.float64, device="cuda")
ht = torch.from_numpy(x)
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(ht, non_blocking=True); torch.cuda.synchronize()
print(f"H2D from registered: {x.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
t = time.perf_counter(); r = cu.cudaHostUnregister(x.ctypes.data)
print(f"cudaHostUnregister: {time.perf_counter()-t:.2f} s rc={r}")
t = time.perf_counter(); d.copy_(ht); torch.cuda.synchronize()
print(f"H2D from pageable (torch): {x.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
for th in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(n), th * 4)
    def cp(c, src=x, dst=pin):
        dst[c[0]:c[-1] + 1] = src[c[0]:c[-1] + 1]
    with ThreadPoolExecutor(th) as pool:
        t = time.perf_counter(); list(pool.map(cp, chunks)); dt = time.perf_counter() - t
    print(f"memcpy pageable->pinned, {th} threads: {x.nbytes/dt/1e9:.1f} GB/s")
