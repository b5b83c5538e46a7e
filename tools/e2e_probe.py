"""Break down BfsEngine.run (the e2e API path) on the bench graph."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_10026_b200 as rb

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
el = rb.kronecker_generate(rb.KroneckerParams(scale=scale), device=True)
g = rb.build_csr(el)
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
eng = rb.BfsEngine(g2, rb.BfsParams())
for r in roots[:3]:
    eng.run(int(r))
T = {"total": [], "traverse": [], "results": [], "host": [], "kernel": []}
for r in roots[:16]:
    r = int(r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eng.run(r)
    T["total"].append(time.perf_counter() - t0)
    T["kernel"].append(res.elapsed_time)
    t0 = time.perf_counter()
    eng._dev.traverse(r)
    t1 = time.perf_counter()
    recs, el_ = eng._dev.results(want_parent=False)
    t2 = time.perf_counter()
    pred = np.empty(g2.n, np.int32)
    eng._dev.parents_to_host(pred)
    t3 = time.perf_counter()
    T["traverse"].append(t1 - t0)
    T["results"].append(t2 - t1)
    T["host"].append(t3 - t2)
for k, v in T.items():
    print(f"{k:9s} median {1e3 * np.median(v):.3f} ms")
for ch in (1, 2, 4, 8, 16):
    ts = []
    for r in roots[:12]:
        eng._dev.traverse(int(r))
        eng._dev.results(want_parent=False)
        t0 = time.perf_counter()
        pred = np.empty(g2.n, np.int32)
        eng._dev.parents_to_host(pred, chunks=ch)
        ts.append(time.perf_counter() - t0)
    print(f"chunks {ch:2d}: host {1e3 * np.median(ts):.3f} ms")
