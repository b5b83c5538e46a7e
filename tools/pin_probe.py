"""D2H rate into (a) an mmap'ed array page-locked with cudaHostRegister (the
result pool), (b) cudaHostAlloc memory (torch pin_memory), before and after the
host's free memory has been churned (what a CPU job before the bench leaves)."""
import ctypes
import mmap
import time

import numpy as np
import torch

N = 32804088
dev = torch.empty(N, dtype=torch.int32, device="cuda")


def rate(host_t, label):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(6):
        t = time.perf_counter()
        host_t.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{label:34s} {4 * N / best / 1e9:6.1f} GB/s")


def registered(nbytes, huge=True):
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if huge:
        m.madvise(mmap.MADV_HUGEPAGE)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    rc = int(torch.cuda.cudart().cudaHostRegister(addr, nbytes, 0))
    a = np.frombuffer(m, dtype=np.int32)
    return m, torch.from_numpy(a), rc


def churn(gb):
    # fragment the free lists: many 1 MB blocks touched, every other one freed, then all freed
    blocks = [np.ones(1 << 18, np.int32) for _ in range(gb * 1024)]
    del blocks[::2]
    big = np.ones(gb * (1 << 27), np.int32)
    del big, blocks


def thp():
    for line in open("/proc/self/smaps_rollup"):
        if line.startswith("AnonHugePages"):
            return line.split()[1] + " kB AnonHugePages"
    return "?"


import sys

for phase in (("now",) if len(sys.argv) > 1 else ("fresh", "after 24 GB churn", "after 48 GB churn")):
    if phase != "fresh":
        churn(24)
    m, t, rc = registered(4 * 67108864)
    t.zero_()
    print(thp())
    rate(t[:N], f"{phase}: mmap + register (rc {rc})")
    m2, t2, rc2 = registered(4 * 67108864, huge=False)
    t2.zero_()
    rate(t2[:N], f"{phase}: mmap 4K pages + register")
    p = torch.empty(67108864, dtype=torch.int32).pin_memory()
    rate(p[:N], f"{phase}: cudaHostAlloc")
    del t, p
