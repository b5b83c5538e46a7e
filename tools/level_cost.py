"""Fixed per-level cost: BFS along a long path (every level = 1 vertex, top-down),
alone and next to a large unreached component (size-dependent per-level work)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_10026_b200 as rb  # noqa: E402

k = 4000
path = np.stack([np.arange(k - 1), np.arange(1, k)], 1).astype(np.uint32)
rng = np.random.default_rng(1)
for extra in ([0, 1 << 22] if len(sys.argv) < 2 else [int(x) for x in sys.argv[1:]]):
    n = k + extra
    e = path
    if extra:
        other = rng.integers(k, n, size=(2 * extra, 2)).astype(np.uint32)
        e = np.concatenate([path, other])
    g = rb.build_csr(rb.EdgeList(n, e))
    with rb.BfsEngine(g, rb.BfsParams()) as eng:
        eng.run_device(0)
        t, levels = eng.run_device(0)
        print(f"path {k} + {extra} unreached: n_dev {eng.n_dev}: {t*1e6/len(levels):.2f} us/level")
        if os.environ.get("RB_DEBUG_TS"):
            import ctypes
            from paper_2012_10026_b200 import _lib
            buf = np.zeros(64 * 4 * 1024, np.uint64)
            nb = ctypes.c_int(0)
            _lib.check(_lib.lib().rb_bfs_debug_timestamps(eng._dev.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size, ctypes.byref(nb)))
            ts = buf[: 64 * 4 * nb.value].reshape(64, nb.value, 4).astype(np.int64)
            for L in range(1, 6):
                a, b, c, dd = ts[L, :, 0], ts[L, :, 1], ts[L, :, 2], ts[L, :, 3]
                an = ts[L + 1, :, 0]
                print(f"  L{L}: counters read {np.median(dd-c)/1e3:.2f} us (max {(dd-c).max()/1e3:.2f}), "
                      f"counters->next start {np.median(an-dd)/1e3:.2f} (max {(an-dd).max()/1e3:.2f})")
                print(f"  L{L}: start skew {(a.max()-a.min())/1e3:.2f} us, work+reduce max {(b-a).max()/1e3:.2f} "
                      f"(median {np.median(b-a)/1e3:.2f}, argmax blk {int(np.argmax(b-a))}), "
                      f"barrier after last arrival {(c.min()-b.max())/1e3:.2f}..{(c.max()-b.max())/1e3:.2f} us, "
                      f"level span {(c.max()-a.min())/1e3:.2f} us")
