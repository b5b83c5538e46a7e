"""CPU oracle for the rcmbfs hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product package ``paper_2012_10026_b200`` never imports it; its kernels are
checked *against* it.

* ``oracle.c`` restates the reference's CSR build, RCM, relabel, sequential /
  hybrid BFS, single steps and validator (file:line cited per function).
* ``kronecker_generate`` below restates ``generator.py:74-148`` with numpy's
  Philox, exactly as the reference does.
* Pinning: ``tests/test_oracle.py`` checks this oracle against the reference's
  own known answers (SCALE10_SEED42_M_DIRECTED = 20922, SCALE16_SEED7 goldens,
  test_graph.py:48-58 worked example, direction patterns of
  test_engine.py:406-420) and against fixtures produced by running the
  reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    """Compile ``liboracle.so`` with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_build_csr.argtypes = [I64, I64, P, P, P, P, P]
        L.or_build_csr.restype = I64
        L.or_degree_sort_rows.argtypes = [I64, P, P, P, P, I32]
        L.or_rcm.argtypes = [I64, P, P, P, P, P, P]
        L.or_rcm.restype = I64
        L.or_apply_permutation.argtypes = [I64, P, P, P, P, P, P, P, P]
        L.or_seq_bfs.argtypes = [I64, P, P, I64, P, P, P, P]
        L.or_seq_bfs.restype = I64
        L.or_td_step.argtypes = [I64, P, P, P, I64, P, P, P, P]
        L.or_bu_step.argtypes = [I64, P, P, P, P, P, P, P]
        L.or_hybrid_bfs.argtypes = [I64, P, P, P, I64, I32, I32, I32, I32, P, P, I64, ctypes.POINTER(D)]
        L.or_hybrid_bfs.restype = I64
        L.or_components.argtypes = [I64, I64, P, I64, P, I64, P]
        L.or_validate.argtypes = [I64, P, P, P, I64, P, P, P]
        L.or_validate.restype = I32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# graph.py:85-120


@dataclass
class Csr:
    n: int
    row_starts: np.ndarray  # int64 (n+1)
    dst: np.ndarray  # uint32
    degrees: np.ndarray  # int32

    @property
    def m_directed(self) -> int:
        return int(self.dst.size)


def build_csr(n: int, edges: np.ndarray) -> Csr:
    e = _c(np.asarray(edges).reshape(-1, 2), np.uint32)
    m = e.shape[0]
    rs = np.zeros(n + 1, np.int64)
    dst = np.empty(max(2 * m, 1), np.uint32)
    deg = np.zeros(max(n, 1), np.int32)
    bad = np.zeros(1, np.int64)
    md = lib().or_build_csr(n, m, _p(e), _p(rs), _p(dst), _p(deg), _p(bad))
    if md < 0:
        i = int(bad[0])
        raise ValueError(f"edge {i} = ({int(e[i, 0])}, {int(e[i, 1])}) out of range for n={n}")
    return Csr(n, rs, dst[:md].copy(), deg[:n].copy())


# ---------------------------------------------------------------------------
# reorder.py


def degree_sort_rows(g: Csr, descending: bool) -> np.ndarray:
    out = np.empty_like(g.dst)
    if g.n:
        lib().or_degree_sort_rows(g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), _p(out), int(descending))
    return out


def rcm(g: Csr):
    """Returns (perm uint32 new->old, n_plus, component_ranges list) -- reorder.py:198-237."""
    perm = np.empty(max(g.n, 1), np.uint32)
    cs = np.empty(g.n + 1, np.int64)
    npl = np.zeros(1, np.int64)
    nc = lib().or_rcm(g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), _p(perm), _p(cs), _p(npl))
    k = int(npl[0])
    bounds = np.append(cs[:nc], k)
    ranges = [(int(k - bounds[i + 1]), int(k - bounds[i])) for i in range(nc - 1, -1, -1)]
    return perm[: g.n].copy(), k, ranges


def inverse(perm: np.ndarray) -> np.ndarray:
    inv = np.empty(perm.size, np.uint32)
    inv[perm] = np.arange(perm.size, dtype=np.uint32)
    return inv


def apply_permutation(g: Csr, perm: np.ndarray) -> Csr:
    perm = _c(perm, np.uint32)
    inv = inverse(perm)
    rs = np.zeros(g.n + 1, np.int64)
    dst = np.empty_like(g.dst)
    deg = np.empty(max(g.n, 1), np.int32)
    if g.n:
        lib().or_apply_permutation(
            g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), _p(perm), _p(inv), _p(rs), _p(dst), _p(deg)
        )
    return Csr(g.n, rs, dst, deg[: g.n].copy())


# ---------------------------------------------------------------------------
# BFS: _kernels.py, engine.py


def seq_bfs(g: Csr, source: int):
    """(parent int32, level int32, n_levels) -- _kernels.py:26-54."""
    parent = np.empty(g.n, np.int32)
    level = np.empty(g.n, np.int32)
    queue = np.empty(g.n, np.uint32)
    bounds = np.empty(g.n + 2, np.int64)
    nl = lib().or_seq_bfs(g.n, _p(g.row_starts), _p(g.dst), int(source), _p(parent), _p(level), _p(queue), _p(bounds))
    return parent, level, int(nl), bounds[: nl + 1].copy()


def hybrid_bfs(g: Csr, source: int, alpha=64, beta=8, hybrid=True, threads=0):
    """Multithreaded restatement of BfsEngine.run mode hybrid/level_sync.

    Returns (parent, records ndarray (L,6): level, dir(0 TD/1 BU), n_f, m_f,
    m_u, scanned; elapsed seconds)."""
    parent = np.empty(g.n, np.int32)
    cap = max(64, g.n + 2)
    rec = np.zeros((min(cap, 1 << 16), 6), np.int64)
    el = ctypes.c_double(0.0)
    nl = lib().or_hybrid_bfs(
        g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), int(source), int(alpha), int(beta),
        int(bool(hybrid)), int(threads), _p(parent), _p(rec), rec.shape[0], ctypes.byref(el),
    )
    return parent, rec[: min(nl, rec.shape[0])].copy(), el.value


def td_step(g: Csr, frontier: np.ndarray, visited_words: np.ndarray, parent: np.ndarray):
    """Sequential td_plain (_kernels.py:57-87); mutates visited/parent."""
    f = _c(frontier, np.uint32)
    nq = np.empty(max(g.n, 1), np.uint32)
    out = np.zeros(3, np.int64)
    lib().or_td_step(g.n, _p(g.row_starts), _p(g.dst), _p(f), f.size, _p(parent), _p(visited_words), _p(nq), _p(out))
    return nq[: out[0]].copy(), out


def bu_step(g: Csr, fcur_words: np.ndarray, visited_words: np.ndarray, parent: np.ndarray):
    """bu_range over [0, n) (_kernels.py:144-173); returns (fnext words, counters)."""
    fnext = np.zeros_like(visited_words)
    out = np.zeros(3, np.int64)
    lib().or_bu_step(g.n, _p(g.row_starts), _p(g.dst), _p(fcur_words), _p(fnext), _p(visited_words), _p(parent), _p(out))
    return fnext, out


# ---------------------------------------------------------------------------
# validate.py


def components(n: int, edges: np.ndarray) -> np.ndarray:
    """Union-find labels (min id root) over raw pairs -- validate.py:63-86."""
    e = _c(np.asarray(edges).reshape(-1, 2), np.uint32)
    root = np.empty(max(n, 1), np.int64)
    lib().or_components(n, e.shape[0], _p(e), 2, _p(e[:, 1:]) if e.shape[0] else _p(e), 2, _p(root))
    return root[:n].copy()


def csr_components(g: Csr) -> np.ndarray:
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_starts))
    return components(g.n, np.stack([src, g.dst], axis=1) if g.n else np.zeros((0, 2), np.uint32))


def validate(g: Csr, labels: np.ndarray, source: int, parent: np.ndarray):
    """Five rules (validate.py:123-225). Returns (passed, ok[5], derived levels int64)."""
    parent = _c(parent, np.int32)
    levels = np.empty(max(g.n, 1), np.int64)
    ok = np.zeros(5, np.int32)
    r = lib().or_validate(g.n, _p(g.row_starts), _p(g.dst), _p(_c(labels, np.int64)), int(source), _p(parent), _p(levels), _p(ok))
    return bool(r), ok.astype(bool), levels[: g.n].copy()


# ---------------------------------------------------------------------------
# generator.py:74-148 (numpy Philox, identical construction)

_M64 = (1 << 64) - 1
CHUNK_EDGES = 1 << 16


def _splitmix64(x: int) -> int:  # generator.py:74-79
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def scramble_constants(scale: int, seed: int):  # generator.py:82-93
    x = (seed ^ 0xD6E8FEB86659FD93) & _M64
    out = []
    shifts = (max(1, scale // 2), max(1, scale // 3), max(1, (2 * scale) // 3))
    for r in range(3):
        x = _splitmix64(x)
        mult = x | 1
        x = _splitmix64(x)
        out.append((mult, x, shifts[r]))
    return out


def scramble_ids(ids, scale: int, seed: int) -> np.ndarray:  # generator.py:96-111
    mask = np.uint64((1 << scale) - 1)
    x = np.asarray(ids, dtype=np.uint64).copy()
    for mult, add, shift in scramble_constants(scale, seed):
        x *= np.uint64(mult & _M64)
        x &= mask
        x ^= x >> np.uint64(shift)
        x += np.uint64(add & ((1 << scale) - 1))
        x &= mask
    return x


def kronecker_generate(scale: int, edgefactor: int = 16, initiator=(0.57, 0.19, 0.19, 0.05), seed: int = 1):
    """(n, edges uint32 (m,2)) -- generator.py:114-148."""
    a, b, c, _ = initiator
    t1, t2, t3 = a, a + b, a + b + c
    n = 1 << scale
    m = n * edgefactor
    out = np.empty((m, 2), dtype=np.uint32)
    weights = np.uint64(1) << np.arange(scale - 1, -1, -1, dtype=np.uint64)
    for chunk, lo in enumerate(range(0, m, CHUNK_EDGES)):
        hi = min(lo + CHUNK_EDGES, m)
        rng = np.random.Generator(np.random.Philox(key=np.array([seed, chunk], dtype=np.uint64)))
        u = rng.random((hi - lo, scale))
        q = (u >= t1).astype(np.uint8) + (u >= t2).astype(np.uint8) + (u >= t3).astype(np.uint8)
        src = ((q >> 1) & 1).astype(np.uint64) @ weights
        dst = (q & 1).astype(np.uint64) @ weights
        out[lo:hi, 0] = scramble_ids(src, scale, seed)
        out[lo:hi, 1] = scramble_ids(dst, scale, seed)
    return n, out


def _mulhi64(x: np.ndarray, t: int) -> np.ndarray:
    """floor(x * t / 2^64) for uint64 x, exact (32-bit limbs)."""
    m32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    xl, xh = x & m32, x >> s32
    tl, th = np.uint64(t & 0xFFFFFFFF), np.uint64(t >> 32)
    p0, p1, p2, p3 = xl * tl, xl * th, xh * tl, xh * th
    mid = (p0 >> s32) + (p1 & m32) + (p2 & m32)
    return p3 + (p1 >> s32) + (p2 >> s32) + (mid >> s32)


def chunglu_generate(n: int, avg_degree: int = 20, gamma: float = 2.1, w_min: float = 1.0, cap_frac: float = 0.01,
                     seed: int = 7):
    """(n, edges uint32 (m,2)): numpy restatement of the Chung-Lu recipe
    (BASELINE configs[4]; no reference generator exists -- the recipe is
    stated in paper_2012_10026_b200/generator.py::ChungLuParams)."""
    rng = np.random.Generator(np.random.Philox(key=np.array([seed, (1 << 32) - 1], dtype=np.uint64)))
    u = rng.random(n)
    cap = float(max(1, int(cap_frac * n)))
    w = np.minimum(cap, w_min * (1.0 - u) ** (-1.0 / (gamma - 1.0)))
    prefix = np.cumsum(np.floor(w * 1024.0).astype(np.int64))
    total = int(prefix[-1])
    m = n * avg_degree // 2
    out = np.empty((m, 2), dtype=np.uint32)
    for chunk, lo in enumerate(range(0, m, CHUNK_EDGES)):
        hi = min(lo + CHUNK_EDGES, m)
        bg = np.random.Philox(key=np.array([seed, (1 << 32) + chunk], dtype=np.uint64))
        raw = bg.random_raw(2 * (hi - lo)).astype(np.uint64)
        r = _mulhi64(raw, total).astype(np.int64)
        out[lo:hi] = np.searchsorted(prefix, r, side="right").reshape(-1, 2).astype(np.uint32)
    return n, out


def sample_sources(degrees: np.ndarray, rounds: int, seed: int) -> np.ndarray:
    """bench.py:124-134."""
    eligible = np.flatnonzero(np.asarray(degrees) > 0)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(eligible, size=rounds, replace=False)).astype(np.int64)
