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
a = ap.parse_args()
import torch  # noqa: E402

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
    eng.run_device(s)
    flush.zero_()
    t, levels = eng.run_device(s)
print(f"root {s} (index {a.index}): {t * 1e6:.1f} us")
for r in levels:
    print(f"  L{r.level} {r.direction[0].upper()}{(r.executed_direction or r.direction)[0].upper()} n_f={r.n_f} "
          f"m_f={r.m_f} scanned={r.scanned_edges} t={r.wall_time * 1e6:.1f} us (phase A {r.queue_time * 1e6:.1f} us)")
