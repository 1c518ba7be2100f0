"""Developer probe: cost of the host-side buffers of a 2,368-field round trip
(9.8 GB): cudaHostAlloc, cudaHostRegister, pageable first touch, and D2H into
page-locked vs pageable memory."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
GB = float(sys.argv[1]) if len(sys.argv) > 1 else 9.83
nbytes = int(GB * 1e9) // 4096 * 4096
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
t = time.perf_counter(); h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); t1 = time.perf_counter()
print(f"cudaHostAlloc {nbytes/1e9:.2f} GB: {t1 - t:.3f} s", flush=True)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d); torch.cuda.synchronize()
    print(f"D2H pinned: {time.perf_counter() - t:.3f} s", flush=True)
del h
t = time.perf_counter(); a = np.empty(nbytes, np.uint8); a[::4096] = 1; t1 = time.perf_counter()
print(f"pageable first touch (1 thread): {t1 - t:.3f} s", flush=True)
t = time.perf_counter(); r = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, nbytes, 0); t1 = time.perf_counter()
print(f"cudaHostRegister: {t1 - t:.3f} s (rc {r})", flush=True)
ta = torch.from_numpy(a)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); ta.copy_(d); torch.cuda.synchronize()
    print(f"D2H registered: {time.perf_counter() - t:.3f} s", flush=True)
torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); ta.copy_(d); torch.cuda.synchronize()
    print(f"D2H pageable (driver staging): {time.perf_counter() - t:.3f} s", flush=True)
b = np.empty(nbytes, np.uint8)
tb = torch.from_numpy(b)
torch.cuda.synchronize(); t = time.perf_counter(); tb.copy_(d); torch.cuda.synchronize()
print(f"D2H pageable fresh (faults): {time.perf_counter() - t:.3f} s", flush=True)
