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
        L.or_build_csr_begin.argtypes = [I64, I64, P, I32, P, ctypes.POINTER(P)]
        L.or_build_csr_begin.restype = I64
        L.or_build_csr_take.argtypes = [P, P, P, P]
        L.or_degree_sort_rows.argtypes = [I64, P, P, P, P, I32]
        L.or_rcm_k.argtypes = [I64, P, P, P, I64, P, P, P]
        L.or_rcm_k.restype = I64
        L.or_apply_permutation.argtypes = [I64, P, P, P, P, P, P, P, P]
        L.or_seq_bfs.argtypes = [I64, P, P, I64, P, P, P, P]
        L.or_seq_bfs.restype = I64
        L.or_td_step.argtypes = [I64, P, P, P, I64, P, P, P, P]
        L.or_bu_step.argtypes = [I64, P, P, P, P, P, P, P]
        L.or_bfs_run.argtypes = [I64, P, P, P, P, I64, I32, I32, I32, I32, I32, P, P, P, I64, ctypes.POINTER(D)]
        L.or_bfs_run.restype = I64
        L.or_get_partitions.argtypes = [I64, I64, I64, P, P]
        L.or_get_partitions.restype = I64
        L.or_shrink_bounds.argtypes = [P, P, P, P]
        U64 = ctypes.c_uint64
        L.or_kronecker_generate.argtypes = [I32, I64, U64, D, D, D, I32, P]
        L.or_chunglu_sample.argtypes = [P, I64, I64, U64, I32, P]
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


def build_csr(n: int, edges: np.ndarray, threads: int = 0) -> Csr:
    """graph.py:85-120 (OpenMP, ``threads`` 0 = all)."""
    e = _c(np.asarray(edges).reshape(-1, 2), np.uint32)
    m = e.shape[0]
    bad = np.zeros(1, np.int64)
    h = ctypes.c_void_p(0)
    md = lib().or_build_csr_begin(n, m, _p(e), int(threads), _p(bad), ctypes.byref(h))
    if md < 0:
        i = int(bad[0])
        raise ValueError(f"edge {i} = ({int(e[i, 0])}, {int(e[i, 1])}) out of range for n={n}")
    rs = np.empty(n + 1, np.int64)
    dst = np.empty(max(md, 1), np.uint32)
    deg = np.empty(max(n, 1), np.int32)
    lib().or_build_csr_take(h, _p(rs), _p(dst), _p(deg))
    return Csr(n, rs, dst[:md], deg[:n])


# ---------------------------------------------------------------------------
# reorder.py


def degree_sort_rows(g: Csr, descending: bool) -> np.ndarray:
    out = np.empty_like(g.dst)
    if g.n:
        lib().or_degree_sort_rows(g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), _p(out), int(descending))
    return out


def rcm(g: Csr, k: int | None = None):
    """Returns (perm uint32 new->old, n_plus, component_ranges list) -- reorder.py:198-237.
    ``k`` labels only (partial_rcm, reorder.py:240-251); ranges then end at k."""
    perm = np.empty(max(g.n, 1), np.uint32)
    cs = np.empty(g.n + 1, np.int64)
    npl = np.zeros(1, np.int64)
    nc = lib().or_rcm_k(g.n, _p(g.row_starts), _p(g.dst), _p(g.degrees), -1 if k is None else int(k), _p(perm),
                        _p(cs), _p(npl))
    k = int(npl[0]) if k is None else min(int(k), int(npl[0]))
    if k == 0:
        return perm[: g.n].copy(), int(npl[0]), []
    bounds = np.append(cs[:nc], k)
    ranges = [(int(k - bounds[i + 1]), int(k - bounds[i])) for i in range(nc - 1, -1, -1)]
    return perm[: g.n].copy(), int(npl[0]), ranges


def partial_rcm(g: Csr, p: float):
    """reorder.py:240-251: the walk stops after ceil(p * |V+|) labels."""
    import math

    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    deg_pos = int(np.count_nonzero(g.degrees > 0))
    return rcm(g, min(math.ceil(p * deg_pos), deg_pos))


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


MODE_CODES = {"level_sync": 0, "hybrid": 1, "hybrid_balanced": 2, "hybrid_reduced": 3}


def bfs_run(g: Csr, source: int, mode: str = "hybrid", alpha=64, beta=8, threads=0, partition_factor=None,
            g_desc_dst: np.ndarray | None = None, want_levels: bool = False):
    """BfsEngine.run (engine.py:518-604) in every mode but "sequential",
    OpenMP with ``threads`` workers (0 = all; = the reference's params.threads,
    so the partition count is partition_factor * threads).

    Returns (parent, levels or None, records ndarray (L, 9): level, dir (0 TD /
    1 BU), n_f, m_f, m_u, scanned, pass1_hits, live_vertices, claimed (-1 =
    None), elapsed seconds)."""
    code = MODE_CODES[mode]
    if code == 3 and g_desc_dst is None:
        g_desc_dst = degree_sort_rows(g, True)
    if threads <= 0:
        threads = os.cpu_count() or 1
    if partition_factor is None:
        partition_factor = 20
    parent = np.empty(max(g.n, 1), np.int32)
    level = np.empty(max(g.n, 1), np.int32) if want_levels else None
    cap = min(max(64, g.n + 2), 1 << 16)
    rec = np.zeros((cap, 9), np.int64)
    el = ctypes.c_double(0.0)
    nl = lib().or_bfs_run(
        g.n, _p(g.row_starts), _p(g.dst), _p(g_desc_dst) if g_desc_dst is not None else None, _p(g.degrees),
        int(source), int(alpha), int(beta), code, int(partition_factor), int(threads), _p(parent),
        _p(level) if level is not None else None, _p(rec), cap, ctypes.byref(el),
    )
    return parent[: g.n], None if level is None else level[: g.n], rec[: min(nl, cap)].copy(), el.value


def hybrid_bfs(g: Csr, source: int, alpha=64, beta=8, hybrid=True, threads=0):
    """mode hybrid (or level_sync): (parent, records (L, 6): level, dir, n_f, m_f, m_u, scanned, elapsed)."""
    parent, _, rec, el = bfs_run(g, source, "hybrid" if hybrid else "level_sync", alpha, beta, threads)
    return parent, rec[:, :6].copy(), el


def get_partitions(n: int, partition_factor: int, threads: int):
    """partition.py:98-140 -> (starts, ends) int64."""
    cap = max(1, partition_factor * threads)
    st = np.empty(cap, np.int64)
    en = np.empty(cap, np.int64)
    k = lib().or_get_partitions(n, partition_factor, threads, _p(st), _p(en))
    return st[:k].copy(), en[:k].copy()


def shrink_bounds(vis_words: np.ndarray, ext_words: np.ndarray, lo: int, hi: int):
    """partition.py:143-171 over uint64 words."""
    a = np.array([lo], np.int64)
    b = np.array([hi], np.int64)
    lib().or_shrink_bounds(_p(_c(vis_words, np.uint64)), _p(_c(ext_words, np.uint64)), _p(a), _p(b))
    return int(a[0]), int(b[0])


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


def kronecker_generate(scale: int, edgefactor: int = 16, initiator=(0.57, 0.19, 0.19, 0.05), seed: int = 1,
                       threads: int = 0):
    """(n, edges uint32 (m,2)) -- generator.py:114-148, C + OpenMP restatement
    (pinned against kronecker_generate_numpy and the reference's hashes)."""
    a, b, c, _ = initiator
    n = 1 << scale
    out = np.empty((n * edgefactor, 2), dtype=np.uint32)
    lib().or_kronecker_generate(scale, edgefactor, seed, float(a), float(b), float(c), int(threads), _p(out))
    return n, out


def kronecker_generate_numpy(scale: int, edgefactor: int = 16, initiator=(0.57, 0.19, 0.19, 0.05), seed: int = 1):
    """(n, edges uint32 (m,2)) -- generator.py:114-148 with numpy's own Philox."""
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
                     seed: int = 7, threads: int = 0):
    """Chung-Lu recipe: weights in numpy (float step), sampling in C + OpenMP
    (pinned against chunglu_generate_numpy)."""
    rng = np.random.Generator(np.random.Philox(key=np.array([seed, (1 << 32) - 1], dtype=np.uint64)))
    u = rng.random(n)
    cap = float(max(1, int(cap_frac * n)))
    w = np.minimum(cap, w_min * (1.0 - u) ** (-1.0 / (gamma - 1.0)))
    prefix = np.cumsum(np.floor(w * 1024.0).astype(np.int64))
    m = n * avg_degree // 2
    out = np.empty((m, 2), dtype=np.uint32)
    lib().or_chunglu_sample(_p(prefix), n, m, seed, int(threads), _p(out))
    return n, out


def chunglu_generate_numpy(n: int, avg_degree: int = 20, gamma: float = 2.1, w_min: float = 1.0,
                           cap_frac: float = 0.01, seed: int = 7):
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
