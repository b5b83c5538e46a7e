"""Distribution of BfsEngine.run wall times (the e2e path) over the 64 bench
roots, three passes, plus the raw D2H copy time of the parents into a
page-locked pooled array -- to see where the e2e outliers come from."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10026_b200 as rb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
el = rb.kronecker_generate(rb.KroneckerParams(scale=scale), device=True)
g = rb.build_csr(el)
del el
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
eng = rb.BfsEngine(g2, rb.BfsParams())
for s in roots[:3]:
    eng.run(int(s))
for p in range(3):
    ts, dev = [], []
    for s in roots:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = eng.run(int(s))
        ts.append(time.perf_counter() - t0)
        dev.append(res.elapsed_time)
    ts = np.array(ts) * 1e3
    print(f"pass {p}: e2e ms min {ts.min():.2f} med {np.median(ts):.2f} max {ts.max():.2f} "
          f"(>1.5x median: {int((ts > 1.5 * np.median(ts)).sum())}); device ms med {1e3 * np.median(dev):.3f}; "
          f"slowest idx {np.argsort(-ts)[:5].tolist()}")
n = eng.n_dev
d = torch.empty(n, dtype=torch.int32, device="cuda")
from paper_2012_10026_b200.engine import fresh_int32  # noqa: E402
a, reg = fresh_int32(g2.n, want_registered=True)
t = torch.from_numpy(a)[:n]
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H {4 * n / 1e6:.0f} MB into {'registered' if reg else 'pageable'}: {dt * 1e3:.2f} ms = {4 * n / dt / 1e9:.1f} GB/s")
