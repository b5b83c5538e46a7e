"""Run ONE bench root (by index into the 64 seeded roots) twice -- warm-up,
then L2 flush + the measured run -- for a targeted ncu capture:
  ncu --set full -k regex:bfs_persistent -s 1 -c 1 python tools/one_root.py --scale 26 --index 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--index", type=int, default=0)
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "chunglu"])
ap.add_argument("--no-warmup", action="store_true", help="profile the first run (ncu flushes caches per replay)")
a = ap.parse_args()
import torch  # noqa: E402

if a.graph == "chunglu":
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << a.scale), device=True)
else:
    el = rb.kronecker_generate(rb.KroneckerParams(scale=a.scale), device=True)
g = rb.build_csr(el)
del el
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
s = int(roots[a.index])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    if not a.no_warmup:
        eng.run_device(s)
    flush.zero_()
    t, levels = eng.run_device(s)
    print(f"root {s} (index {a.index}): {t * 1e6:.1f} us")
    for r in levels:
        print(f"  L{r.level} {r.direction[0].upper()}{(r.executed_direction or r.direction)[0].upper()} n_f={r.n_f} "
              f"m_f={r.m_f} scanned={r.scanned_edges} t={r.wall_time * 1e6:.1f} us (phase A {r.queue_time * 1e6:.1f} us)")
    if os.environ.get("RB_DEBUG_TS"):  # CTA 0 sub-phase stamps of each grid level (solo levels excluded)
        import ctypes

        import numpy as np
        from paper_2012_10026_b200 import _lib

        buf = np.zeros(65536 + 64 * 148 * 32, np.uint64)
        nb = ctypes.c_int(0)
        _lib.check(_lib.lib().rb_bfs_debug_timestamps(eng._dev.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                                      ctypes.byref(nb)))
        ts = buf[: 64 * 4 * nb.value].reshape(64, nb.value, 4).astype(np.int64)
        ph = buf[60000: 60000 + 64 * 8].reshape(64, 8).astype(np.int64)
        ent, ext = int(ph[63, 0]), int(ph[63, 1])
        lev_sum = sum(r.wall_time for r in levels)
        print(f"  kernel entry->exit {(ext - ent) / 1e3:.1f} us (CTA 0), sum of level times {lev_sum * 1e6:.1f} us, "
              f"event time {t * 1e6:.1f} us")
        for L in range(len(levels)):
            t0 = ts[L, 0, 0]
            if t0 == 0:
                continue
            marks = " ".join(f"p{j}={(ph[L, j] - t0) / 1e3:.1f}" for j in range(8) if ph[L, j] > t0)
            print(f"  stamps L{L}: work end {(ts[L, 0, 1] - t0) / 1e3:.1f} us  {marks}")
            if L + 1 < 64 and ph[L + 1, 5] > t0:  # a solo tail entered after this level
                print(f"    tail entry after L{L}: " + " ".join(f"p{j}={(ph[L + 1, j] - t0) / 1e3:.1f}" for j in (5, 6, 7)))
                wt = buf[65536 + (L + 1) * nb.value * 32: 65536 + (L + 2) * nb.value * 32].astype(np.int64)
                wt = (wt - t0) / 1e3
                order = np.argsort(-wt)[:8]
                print("    slowest warps (cta, warp, end us):", [(int(i // 32), int(i % 32), round(float(wt[i]), 1)) for i in order])
                raw = buf[65536 + (L + 1) * nb.value * 32: 65536 + (L + 2) * nb.value * 32]
                print("    warps without a stamp:", int((raw == 0).sum()), "of", raw.size, " min end", round(float(wt.min()), 1))
