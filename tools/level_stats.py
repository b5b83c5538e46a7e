"""Per-level-index statistics over the 64 bench roots (L2 flushed before each):
mean device time, labelled/executed direction mix, mean n_f / m_f / scanned.
RB_LIB selects a library variant (A/B on one box).

  python tools/level_stats.py [--scale 26] [--graph kronecker|chunglu] [--roots 64]
"""
import argparse
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "chunglu"])
ap.add_argument("--roots", type=int, default=64)
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
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)[: a.roots]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
agg = collections.defaultdict(list)
tot = []
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    for s in roots[:3]:
        eng.run_device(int(s))
    slow = []
    for i, s in enumerate(roots):
        flush.zero_()
        t, levels = eng.run_device(int(s))
        tot.append(t)
        slow.append((t, i, "".join(r.direction[0].upper() + (r.executed_direction or r.direction)[0].upper() + " "
                                   for r in levels)))
        reached = 0
        for r in levels:
            reached += r.n_f
            r.unvisited = st.n_non_isolated - reached  # before the level's discoveries
            agg[r.level].append(r)
for t, i, d in sorted(slow)[-6:]:
    print(f"slow root index {i}: {1e6 * t:.1f} us  {d}")
print(f"{os.environ.get('RB_LIB', 'in-tree')}: mean {1e6 * np.mean(tot):.1f} us/root over {len(tot)} roots")
for L in sorted(agg):
    rs = agg[L]
    mix = collections.Counter(r.direction[0].upper() + ((r.executed_direction or r.direction)[0].upper()) for r in rs)
    t = np.array([r.wall_time for r in rs]) * 1e6
    imax = int(np.argmax(t))
    print(f"  L{L:<2d} n={len(rs):2d} {dict(mix)}  t mean {t.mean():7.1f} max {t.max():7.1f} us | "
          f"n_f {np.mean([r.n_f for r in rs]):11.0f} m_f {np.mean([r.m_f for r in rs]):12.0f} "
          f"scanned {np.mean([r.scanned_edges for r in rs]):11.0f}  sum/64 {t.sum() / len(tot):6.1f}"
          f"  | max: n_f {rs[imax].n_f} m_f {rs[imax].m_f}")
    for k in sorted(mix):
        sel = [r for r in rs if r.direction[0].upper() + ((r.executed_direction or r.direction)[0].upper()) == k]
        tk = [r.wall_time * 1e6 for r in sel]
        print(f"       {k}: n={len(tk):2d} t mean {np.mean(tk):7.1f} us  n_f {np.mean([r.n_f for r in sel]):11.0f} "
              f"m_f {np.mean([r.m_f for r in sel]):12.0f} m_u {np.mean([r.m_u for r in sel]):12.0f} "
              f"U {np.mean([r.unvisited for r in sel]):11.0f} scanned {np.mean([r.scanned_edges for r in sel]):11.0f}")
