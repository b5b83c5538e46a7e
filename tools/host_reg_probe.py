"""Result-array strategies for the e2e path: hugepage mmap arrays, first touch,
cudaHostRegister / Unregister, DMA straight into a registered array."""
import mmap
import time

import numpy as np
import torch

cudart = torch.cuda.cudart()


def huge_array(n):
    m = mmap.mmap(-1, 4 * n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=np.int32)


for n in (2395985, 4194304, 32804088, 67108864):
    dev = torch.zeros(n, dtype=torch.int32, device="cuda")
    r = {}
    for it in range(3):
        t0 = time.perf_counter(); a = huge_array(n); t1 = time.perf_counter()
        torch.from_numpy(a).fill_(-1); t2 = time.perf_counter()
        r.setdefault("huge alloc", []).append(t1 - t0); r.setdefault("huge first fill (torch)", []).append(t2 - t1)
        b = huge_array(n)
        t0 = time.perf_counter()
        e = cudart.cudaHostRegister(b.ctypes.data, 4 * n, 0)
        t1 = time.perf_counter()
        torch.from_numpy(b).copy_(dev, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
        cudart.cudaHostUnregister(b.ctypes.data); t3 = time.perf_counter()
        r.setdefault(f"register (untouched) rc={int(e)}", []).append(t1 - t0)
        r.setdefault("DMA into registered", []).append(t2 - t1)
        r.setdefault("unregister", []).append(t3 - t2)
        c = np.empty(n, np.int32)
        t0 = time.perf_counter(); e = cudart.cudaHostRegister(c.ctypes.data, 4 * n, 0); t1 = time.perf_counter()
        cudart.cudaHostUnregister(c.ctypes.data); t2 = time.perf_counter()
        r.setdefault("register np.empty", []).append(t1 - t0); r.setdefault("unregister np.empty", []).append(t2 - t1)
    print(f"n={n} ({4 * n / 1e6:.1f} MB)")
    for k, v in r.items():
        print(f"   {k:32s} {1e3 * min(v):8.3f} ms  ({4 * n / min(v) / 1e9:6.1f} GB/s)")
