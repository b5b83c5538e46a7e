"""Where BfsEngine.run's time goes at the bench config: the whole call, the
device traversal, the parents' DMA into a page-locked result array, and the
host fill of the isolated tail (each alone, median of 12 roots)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_10026_b200 as rb
import ctypes

from paper_2012_10026_b200 import _lib, engine

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
el = rb.kronecker_generate(rb.KroneckerParams(scale=scale), device=True)
g = rb.build_csr(el)
del el
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
eng = rb.BfsEngine(g2, rb.BfsParams())
for r in roots[:4]:
    res = eng.run(int(r))
n, n_dev = g2.n, eng.n_dev
T = {"run": [], "kernel": [], "traverse+sync": [], "dma": [], "fill": [], "fresh": []}
keep = []
for r in roots[:12]:
    r = int(r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eng.run(r)
    T["run"].append(time.perf_counter() - t0)
    T["kernel"].append(res.elapsed_time)
    del res
    t0 = time.perf_counter()
    eng._dev.traverse(r)
    torch.cuda.synchronize()
    T["traverse+sync"].append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    pred, reg = engine.fresh_int32(n, want_registered=True)
    T["fresh"].append(time.perf_counter() - t0)
    pt = torch.from_numpy(pred)
    dev = eng.parent_device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pt[:n_dev].copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    T["dma"].append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    pt[n_dev:].fill_(-1)
    T["fill"].append(time.perf_counter() - t0)
    for th in (2, 4, 8, 16):
        t0 = time.perf_counter()
        _lib.lib().rb_host_fill_i32(ctypes.c_void_p(pred.ctypes.data + 4 * n_dev), n - n_dev, -1, th)
        T.setdefault(f"stream fill x{th}", []).append(time.perf_counter() - t0)
    del pt, pred
# the steps of _DeviceBfs.run_to_host, timed on the host
d = eng._dev
L = _lib.lib()
S = {}
for r in roots[:12]:
    r = int(r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.traverse(r)
    t1 = time.perf_counter()
    pred, reg = engine.fresh_int32(n, want_registered=True)
    _lib.check(L.rb_bfs_results_async(d.h, _lib.ptr(d._state), _lib.ptr(d._recs_pin), 64, ctypes.c_void_p(pred.ctypes.data),
                                      1, _lib.stream_ptr()), "async")
    t2 = time.perf_counter()
    L.rb_host_fill_i32(ctypes.c_void_p(pred.ctypes.data + 4 * n_dev), n - n_dev, -1, 8)
    t3 = time.perf_counter()
    L.rb_bfs_wait(d.h, -1)
    t4 = time.perf_counter()
    L.rb_bfs_wait(d.h, 0)
    t5 = time.perf_counter()
    for k, v in (("traverse enqueue", t1 - t0), ("results enqueue", t2 - t1), ("fill", t3 - t2), ("wait state", t4 - t3),
                 ("wait parents", t5 - t4), ("sum", t5 - t0)):
        S.setdefault(k, []).append(v)
    del pred
for k, v in S.items():
    print(f"  step {k:18s} median {1e3 * np.median(v):.3f} ms")
print(f"n {n} n_dev {n_dev} registered {reg} torch threads {torch.get_num_threads()}")
for k, v in T.items():
    print(f"{k:14s} median {1e3 * np.median(v):.3f} ms")
print(f"dma rate {4 * n_dev / np.median(T['dma']) / 1e9:.1f} GB/s, fill rate {4 * (n - n_dev) / np.median(T['fill']) / 1e9:.1f} GB/s")
