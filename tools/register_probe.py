"""Zero-copy feasibility probe for file sources: mmap an SSTATBIN-sized file in /dev/shm,
cudaHostRegister the mapping, and time H2D copies straight from it (vs a pinned buffer).
    python tools/register_probe.py [GB]"""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
nbytes = int(gb * 1e9) // 4096 * 4096
path = "/dev/shm/register_probe.bin"
with open(path, "wb") as f:
    chunk = os.urandom(1 << 20) * 64
    left = nbytes
    while left > 0:
        f.write(chunk[:min(left, len(chunk))])
        left -= len(chunk)
torch.cuda.init()
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is None:
    import glob
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so.*"))
    cudart = ctypes.CDLL(cands[0])
fd = os.open(path, os.O_RDWR)
mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)

arr = np.frombuffer(mm, dtype=np.uint8)
addr = arr.ctypes.data
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for flags in (0x08 | 0x01, 0x01, 0x00):  # ReadOnly|Portable, Portable, default
    t0 = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(addr), ctypes.c_size_t(nbytes), ctypes.c_uint(flags))
    t1 = time.perf_counter()
    print(f"register {nbytes / 1e9:.1f} GB flags={flags}: rc={rc} in {t1 - t0:.3f} s", flush=True)
    if rc == 0:
        break
    cudart.cudaGetLastError()
if rc == 0:
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc2 = cudart.cudaMemcpy(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(addr), ctypes.c_size_t(nbytes), 1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"H2D from registered mapping: rc={rc2} {nbytes / dt / 1e9:.1f} GB/s", flush=True)
    t0 = time.perf_counter()
    cudart.cudaHostUnregister(ctypes.c_void_p(addr))
    print(f"unregister {time.perf_counter() - t0:.3f} s", flush=True)
pin = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D from pinned: {nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
del arr
mm.close()
os.close(fd)
os.remove(path)
