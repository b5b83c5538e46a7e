"""Per root: the first level labelled bottom-up -- n_f, m_f, m_u, executed
direction and device time (for the early executed-direction rule).
  RB_EXEC_ALPHA=1 / 1000000000 python tools/early_dump.py --scale 26"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--graph", default="kronecker")
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tot = 0.0
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    eng.run_device(int(roots[0]))
    for i, s in enumerate(roots):
        flush.zero_()
        t, levels = eng.run_device(int(s))
        tot += t
        for r in levels:
            if r.direction == rb.BOTTOM_UP:
                print(f"root {i:2d} L{r.level} n_f {r.n_f:9d} m_f {r.m_f:11d} m_u {r.m_u:11d} "
                      f"exec {(r.executed_direction or r.direction)[0].upper()} t {r.wall_time * 1e6:8.1f} us  "
                      f"root total {t * 1e6:8.1f}")
                break
print(f"mean {tot / len(roots) * 1e6:.1f} us/root")
