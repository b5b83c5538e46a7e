import sys, time, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_10026_b200 as rb
from paper_2012_10026_b200 import _lib, engine
scale = int(sys.argv[1])
if len(sys.argv) > 2 and sys.argv[2] == "chunglu":
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << scale), device=True)
else:
    el = rb.kronecker_generate(rb.KroneckerParams(scale=scale), device=True)
g = rb.build_csr(el); perm, st = rb.rcm(g); g2 = rb.apply_permutation(g, perm)
roots = rb.sample_sources(g2.device_arrays()[2].cpu().numpy(), 64, 1)
eng = rb.BfsEngine(g2, rb.BfsParams())
for r in roots[:3]: eng.run(int(r))
d = eng._dev
T = {}
def tick(k, t0):
    t = time.perf_counter(); T.setdefault(k, []).append(t - t0); return t
for r in roots[:16]:
    torch.cuda.synchronize()
    t = time.perf_counter(); t00 = t
    res = eng.run(int(r)); t = tick("run total", t)
    # manual breakdown
    L = _lib.lib(); s = _lib.stream_ptr()
    t = time.perf_counter()
    d.traverse(int(r)); t = tick("traverse", t)
    n_dev = d.n_dev; chunks = 4 if n_dev >= (8 << 20) else 2
    _lib.check(L.rb_bfs_results_async(d.h, _lib.ptr(d._state), _lib.ptr(d._recs_pin), 64, _lib.ptr(d.pinned), chunks, s)); t = tick("enqueue copies", t)
    pred = engine.fresh_int32(g2.n); pt = torch.from_numpy(pred); pt[n_dev:].fill_(-1); t = tick("alloc+tail", t)
    L.rb_bfs_wait(d.h, -1); t = tick("wait small", t)
    nrec = ctypes.c_int64(0); L.rb_bfs_complete(d.h, _lib.ptr(d._state), _lib.ptr(d._recs_pin), 64, ctypes.byref(nrec)); t = tick("complete", t)
    step = -(-n_dev // chunks)
    for i in range(chunks):
        a, b = i * step, min((i + 1) * step, n_dev); L.rb_bfs_wait(d.h, i); pt[a:b].copy_(d.pinned[a:b])
    t = tick("chunks", t)
    lv = engine._records_to_levels((_lib.LevelRecordC * nrec.value).from_buffer_copy(d._recs_pin.numpy().tobytes()[: nrec.value * 80])); t = tick("records->levels", t)
print(f"n={g2.n} n_dev={d.n_dev}")
for k, v in T.items(): print(f"{k:18s} {1e3*np.median(v):8.3f} ms")
