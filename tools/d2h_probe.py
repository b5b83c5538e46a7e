"""Host-side cost of returning an n-vertex predecessor array (e2e path), steady state."""
import time

import numpy as np
import torch

n, n_dev = 4194304, 2395985
d = torch.randint(0, 100, (n_dev,), dtype=torch.int32, device="cuda")
pin = torch.empty(n_dev, dtype=torch.int32, pin_memory=True)
print("threads", torch.get_num_threads(), flush=True)


def pageable():
    pred = np.empty(n, np.int32)
    torch.from_numpy(pred)[:n_dev].copy_(d)
    pred[n_dev:] = -1
    return pred


def pinned_torch():
    pin.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    pred = np.empty(n, np.int32)
    pt = torch.from_numpy(pred)
    pt[:n_dev].copy_(pin)
    pt[n_dev:].fill_(-1)
    return pred


def pinned_np():
    pin.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    pred = np.empty(n, np.int32)
    pred[:n_dev] = pin.numpy()
    pred[n_dev:] = -1
    return pred


for f in (pageable, pinned_torch, pinned_np, pageable, pinned_torch):
    ts = []
    r = None
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t0)
    print(f.__name__, " ".join(f"{1e3*x:.2f}" for x in ts), flush=True)
