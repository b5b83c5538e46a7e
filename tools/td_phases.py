"""Per-warp end times of top-down phase A / phase B / level work for one root
(RB_DEBUG_TS=1): where a top-down level's time goes and how uneven the warps are.
  python tools/td_phases.py --index 7 [--scale 26]"""
import argparse
import ctypes
import os
import sys

import numpy as np

os.environ["RB_DEBUG_TS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402
from paper_2012_10026_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--index", type=int, nargs="*", default=[7])
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "chunglu"])
a = ap.parse_args()
import torch  # noqa: E402

if a.graph == "chunglu":
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << a.scale), device=True)
else:
    el = rb.kronecker_generate(rb.KroneckerParams(scale=a.scale), device=True)
g = rb.build_csr(el)
del el
perm, _ = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
KW = 24
WA = 65536 + 0
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    for i in a.index:
        s = int(roots[i])
        eng.run_device(s)
        flush.zero_()
        t, levels = eng.run_device(s)
        buf = np.zeros(65536 + 64 * 1024 * KW, np.uint64)
        nb = ctypes.c_int(0)
        _lib.check(_lib.lib().rb_bfs_debug_timestamps(eng._dev.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                                      ctypes.byref(nb)))
        B = nb.value
        ts = buf[: 64 * 4 * B].reshape(64, B, 4).astype(np.int64)
        ph = buf[60000: 60000 + 64 * 8].reshape(64, 8).astype(np.int64)
        reg = [65536, 65536 + 64 * 256 * 32, 65536 + 2 * 64 * 256 * 32]
        print(f"root {s} (index {i}): {t * 1e6:.1f} us")
        n_solo = len(levels) - int((ts[:, 0, 0] > 0).sum())
        for L, r in enumerate(levels):
            t0 = ts[L, :, 0].min()
            if ts[L, 0, 0] == 0:
                continue
            ex = (r.executed_direction or r.direction)[0].upper()
            line = f"  L{r.level} {r.direction[0].upper()}{ex} n_f={r.n_f} m_f={r.m_f} t={r.wall_time * 1e6:.1f} us"
            marks = " ".join(f"p{j}={(ph[L, j] - t0) / 1e3:.1f}" for j in range(5) if ph[L, j] > t0)
            print(line + "  " + marks)
            if ex != "T":
                continue
            for name, base in zip(("phaseA end", "phaseB end", "work end"), (reg[1], reg[2], reg[0])):
                w = buf[base + L * B * KW: base + (L + 1) * B * KW].astype(np.int64)
                w = w[w > t0]
                if w.size == 0:
                    continue
                w = (w - t0) / 1e3
                print(f"     {name:10s}: warps {w.size:5d} min {w.min():7.1f} p10 {np.percentile(w, 10):7.1f} med {np.median(w):7.1f} "
                      f"p90 {np.percentile(w, 90):7.1f} p99 {np.percentile(w, 99):7.1f} max {w.max():7.1f} us")
