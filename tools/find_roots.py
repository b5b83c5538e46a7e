"""Indices (into the 64 bench roots) whose level sequence contains a given
labelled+executed direction pair at a level, e.g. L2 'BT' (labelled
bottom-up, executed top-down): python tools/find_roots.py --scale 26 --level 2 --kind BT"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--graph", default="kronecker")
ap.add_argument("--level", type=int, default=2)
ap.add_argument("--kind", default="BT")
a = ap.parse_args()
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
hits = []
with rb.BfsEngine(g2, rb.BfsParams()) as eng:
    for i, s in enumerate(roots):
        _, levels = eng.run_device(int(s))
        kinds = [r.direction[0].upper() + (r.executed_direction or r.direction)[0].upper() for r in levels]
        if len(kinds) > a.level and kinds[a.level] == a.kind:
            hits.append(i)
print(" ".join(map(str, hits)))
