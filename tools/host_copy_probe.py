"""Host-side costs of the e2e result path: fresh numpy allocation + first touch,
pinned -> pageable copies (torch / numpy), pinned DMA.  python tools/host_copy_probe.py"""
import time

import numpy as np
import torch

for n in (4194304, 2395985, 32804088, 67108864):
    pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
    dev = torch.zeros(n, dtype=torch.int32, device="cuda")
    res = {}
    for it in range(3):
        t0 = time.perf_counter(); a = np.empty(n, np.int32); t1 = time.perf_counter()
        a.fill(-1); t2 = time.perf_counter()
        res.setdefault("empty", []).append(t1 - t0); res.setdefault("fill(first touch)", []).append(t2 - t1)
        t0 = time.perf_counter(); a.fill(0); t1 = time.perf_counter(); res.setdefault("fill(warm)", []).append(t1 - t0)
        b = np.empty(n, np.int32)
        t0 = time.perf_counter(); torch.from_numpy(b).copy_(pinned); t1 = time.perf_counter()
        res.setdefault("torch copy pinned->fresh", []).append(t1 - t0)
        t0 = time.perf_counter(); torch.from_numpy(b).copy_(pinned); t1 = time.perf_counter()
        res.setdefault("torch copy pinned->warm", []).append(t1 - t0)
        c = np.empty(n, np.int32)
        t0 = time.perf_counter(); np.copyto(c, pinned.numpy()); t1 = time.perf_counter()
        res.setdefault("np.copyto pinned->fresh", []).append(t1 - t0)
        torch.cuda.synchronize()
        t0 = time.perf_counter(); pinned.copy_(dev, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
        res.setdefault("D2H pinned DMA", []).append(t1 - t0)
        d = np.empty(n, np.int32)
        t0 = time.perf_counter(); torch.from_numpy(d).copy_(dev); t1 = time.perf_counter()
        res.setdefault("D2H into fresh pageable", []).append(t1 - t0)
    print(f"n={n} ({4 * n / 1e6:.1f} MB), torch threads {torch.get_num_threads()}")
    for k, v in res.items():
        print(f"   {k:28s} {1e3 * min(v):8.3f} ms  ({4 * n / min(v) / 1e9:6.1f} GB/s)")
