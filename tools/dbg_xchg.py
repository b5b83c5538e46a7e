"""Debug helper: the emulated device-exchange path step by step."""
import sys
import traceback

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2012_10026_b200 as rb  # noqa: E402
from paper_2012_10026_b200 import _lib  # noqa: E402
from paper_2012_10026_b200.distributed import DevicePartition, connect_emulated, partition_bounds, run_emulated  # noqa: E402

el = rb.kronecker_generate(rb.KroneckerParams(scale=16, seed=1), device=True)
g = rb.build_csr(el)
perm, st = rb.rcm(g)
g2 = rb.apply_permutation(g, perm)
torch.cuda.synchronize()
bounds = partition_bounds(g2.row_starts, st.n_non_isolated, 2, 128)
print("bounds", bounds, flush=True)
parts = []
for r in range(2):
    try:
        parts.append(DevicePartition(g2, bounds, r, 2, record_levels=True))
        torch.cuda.synchronize()
        print("part", r, "ok", flush=True)
    except Exception:
        traceback.print_exc()
connect_emulated(parts)
for p in parts:
    try:
        p.reset(3, int(g2.degrees[3]))
        torch.cuda.synchronize()
        print("reset ok", flush=True)
    except Exception:
        traceback.print_exc()
try:
    print(run_emulated(parts, 3, int(g2.degrees[3]))[0][:3])
except Exception:
    traceback.print_exc()
