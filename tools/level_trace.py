"""Per-level device trace of a few roots (direction, n_f, scanned, t_us).

  python tools/level_trace.py [--scale 22] [--roots 4] [--mode hybrid]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "chunglu"])
ap.add_argument("--roots", type=int, default=4)
ap.add_argument("--mode", default="hybrid")
ap.add_argument("--brief", action="store_true")
ap.add_argument("--sources", type=int, nargs="*", default=None)
ap.add_argument("--flush", action="store_true", help="write 256 MiB before each root (cold L2, like bench.py)")
a = ap.parse_args()
if a.graph == "chunglu":
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << a.scale), device=True)
else:
    el = rb.kronecker_generate(rb.KroneckerParams(scale=a.scale), device=True)
g = rb.build_csr(el)
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
with rb.BfsEngine(g2, rb.BfsParams(mode=a.mode)) as eng:
    import ctypes
    from paper_2012_10026_b200 import _lib
    ns = ctypes.c_double(0)
    blocks, threads = ctypes.c_int(0), ctypes.c_int(0)
    _lib.lib().rb_bfs_grid(eng._dev.h, ctypes.byref(blocks), ctypes.byref(threads))
    for it in (10, 1000):
        _lib.check(_lib.lib().rb_bfs_barrier_probe(eng._dev.h, it, ctypes.byref(ns), _lib.stream_ptr()))
        print(f"grid {blocks.value}x{threads.value}: barrier {ns.value:.0f} ns (iters={it})")
    eng.run_device(int(roots[0]))
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for s in (a.sources if a.sources else roots[: a.roots]):
        if a.flush:
            flush.zero_()
        el_s, levels = eng.run_device(int(s))
        print(f"root {s}: {el_s*1e6:.1f} us, levels {len(levels)}  " + " ".join(
            f"{r.direction[0].upper()}{'' if (r.executed_direction or r.direction) == r.direction else '>' + r.executed_direction[0].upper()}{r.wall_time*1e6:.0f}" for r in levels))
        if a.brief:
            continue
        for r in levels:
            x = "" if (r.executed_direction or r.direction) == r.direction else ">" + r.executed_direction[0].upper()
            print(f"   L{r.level} {r.direction[:1].upper()}{x} n_f={r.n_f:9d} m_f={r.m_f:11d} scanned={r.scanned_edges:11d} t={r.wall_time*1e6:8.1f}us (queue {r.queue_time*1e6:6.1f})")
