"""Where do the edges of a deferred top-down level point?  For one bench root: the
level-L frontier's targets binned by id -- the share that falls into the top W ids
(RCM puts the hubs last), first-touch vs duplicate, and already-visited targets.
  python tools/td_skew.py --scale 26 --index 23 --level 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--index", type=int, nargs="*", default=[23])
ap.add_argument("--level", type=int, default=2)
a = ap.parse_args()
import torch  # noqa: E402

el = rb.kronecker_generate(rb.KroneckerParams(scale=a.scale), device=True)
g = rb.build_csr(el)
del el
perm, _ = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
del g, perm
rs, col, deg = g2.device_arrays()[:3]
roots = rb.sample_sources(deg.cpu().numpy(), 64, 1)
n = int(deg.numel())
# degree-weighted share of the top-W ids over the whole graph
cs = torch.cumsum(deg.to(torch.int64), 0)
tot = int(cs[-1])
nd = int((deg > 0).nonzero().max()) + 1
print(f"n {n} n_dev {nd} m {tot}")
for W in (1 << 14, 1 << 16, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
    print(f"  all edges: top {W} ids hold {1 - int(cs[nd - W - 1]) / tot:.3f} of the endpoints")
with rb.BfsEngine(g2, rb.BfsParams(), record_levels=True) as eng:
    for i in a.index:
        s = int(roots[i])
        eng.run_device(s)
        lev = eng.level_device().to(torch.int64)[:nd]
        for L in range(1, 4):
            f = (lev == L).nonzero().flatten()
            d = deg[f].to(torch.int64)
            m = int(d.sum())
            if m == 0 or m > (1 << 28):
                continue
            starts = rs[f]
            offs = torch.cumsum(d, 0) - d
            idx = torch.arange(m, device="cuda") - torch.repeat_interleave(offs, d) + torch.repeat_interleave(starts, d)
            t = col[idx].to(torch.int64)
            del idx
            tl = lev[t]
            new = int((tl == L + 1).sum())
            uniq = int(torch.unique(t[tl == L + 1]).numel())
            print(f"root index {i} level {L}: rows {f.numel()} edges {m}; targets at L+1 {new} ({uniq} distinct), "
                  f"already visited {m - new}")
            for W in (1 << 14, 1 << 16, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
                inw = t >= nd - W
                print(f"    top {W:8d} ids: {int(inw.sum()) / m:.3f} of the edges; of the L+1 edges "
                      f"{int((inw & (tl == L + 1)).sum()) / max(new, 1):.3f}; distinct new in window "
                      f"{int(torch.unique(t[inw & (tl == L + 1)]).numel())}")
            del t, tl
