"""Per-level CTA work-time spread (RB_DEBUG_TS=1): how unevenly a level's work
lands on the 148 CTAs.  python tools/block_skew.py [scale] [graph]"""
import ctypes
import os
import sys

import numpy as np

os.environ["RB_DEBUG_TS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402
from paper_2012_10026_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
if len(sys.argv) > 2 and sys.argv[2] == "chunglu":
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << scale), device=True)
else:
    el = rb.kronecker_generate(rb.KroneckerParams(scale=scale), device=True)
g = rb.build_csr(el)
perm, _ = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g, el
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    idx = [int(x) for x in os.environ.get("RB_ROOT_INDEX", "0,1").split(",")]
    for r in [roots[i] for i in idx]:
        eng.run_device(int(r))
        t, levels = eng.run_device(int(r))
        buf = np.zeros(65536 + 64 * 148 * 32, np.uint64)
        nb = ctypes.c_int(0)
        _lib.check(_lib.lib().rb_bfs_debug_timestamps(eng._dev.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                                      ctypes.byref(nb)))
        ts = buf[: 64 * 4 * nb.value].reshape(64, nb.value, 4).astype(np.int64)
        wt = buf[65536: 65536 + 64 * nb.value * 32].reshape(64, nb.value, 32).astype(np.int64)
        print(f"root {int(r)}: {t * 1e6:.1f} us  (level index L of the debug stamps counts grid levels only)")
        for L, rec in enumerate(levels):
            a, b, c = ts[L, :, 0], ts[L, :, 1], ts[L, :, 2]
            w = (b - a) / 1e3
            print(f"  L{L} {'T' if rec.direction == rb.TOP_DOWN else 'B'} n_f={rec.n_f:>9d}: work+reduce "
                  f"min {w.min():7.1f} med {np.median(w):7.1f} p90 {np.percentile(w, 90):7.1f} max {w.max():7.1f} us"
                  f" | span {(c.max() - a.min()) / 1e3:7.1f} us")
            ww = (wt[L] - a[:, None]) / 1e3  # per-warp end of work, from its CTA's level start
            inner = ww.max(axis=1) - ww.mean(axis=1)
            print(f"       warps: mean end {ww.mean():7.1f}  mean(CTA max - CTA mean) {inner.mean():6.1f} us"
                  f"  grid max {ww.max():7.1f}")
