"""1D-partition BFS: the exchange / policy driver over
world_size-2 gloo on CPU with a numpy local step, checked against the oracle
(levels bit-exact, level records identical, parent trees valid).  The GPU
local step is exercised by tests/test_gpu_distributed.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2012_10026_b200.distributed import ALIGN, PartitionedBfs, partition_bounds, words_for


def test_partition_bounds_balanced_and_aligned():
    rng = np.random.default_rng(0)
    for n, world, align in ((100_000, 4, 8192), (50_000, 8, 256), (10, 3, 32), (4096, 2, 8192)):
        deg = rng.integers(0, 50, size=n) * (np.arange(n) / n > 0.5)  # skewed: heavy tail at high ids
        rs = np.zeros(n + 1, np.int64)
        np.cumsum(deg, out=rs[1:])
        b = partition_bounds(rs, n, world, align)
        assert b[0] == 0 and b[-1] == n and len(b) == world + 1
        assert all(x <= y for x, y in zip(b, b[1:]))
        assert all(x % align == 0 for x in b[:-1])
        if n >= world * align * 4:
            w = rs[np.array(b[1:])] - rs[np.array(b[:-1])] + np.diff(b)
            assert w.max() <= 1.5 * w.sum() / world + align * 60


class CpuLocalLevel:
    """numpy restatement of one rank's partitioned level (test infrastructure)."""

    device = torch.device("cpu")

    def __init__(self, g, bounds, rank):
        self.g = g
        self.lo, self.hi = bounds[rank], bounds[rank + 1]
        self.n_local = self.hi - self.lo
        rs = g.row_starts
        # transpose slice: owned neighbours of every global vertex
        self.tr = [[] for _ in range(bounds[-1])]
        for w in range(self.lo, self.hi):
            for u in g.dst[rs[w] : rs[w + 1]]:
                self.tr[int(u)].append(w)
        self.n_words_local = words_for(max(self.n_local, 1))

    def reset(self, source):
        self.vis = self.g.degrees[self.lo : self.hi] == 0
        self.parent = np.full(self.n_local, -1, np.int64)
        if self.lo <= source < self.hi:
            self.vis[source - self.lo] = True
            self.parent[source - self.lo] = source

    def make_nz(self, glob):
        return None

    def level(self, L, direction, hubs, glob, nz):
        bits = np.unpackbits(glob.numpy().view(np.uint8), bitorder="little").astype(bool)
        nxt = np.zeros(self.n_local, bool)
        deg_next = maxdeg = scanned = 0
        g = self.g
        if direction == 0:
            for u in np.flatnonzero(bits[: len(self.tr)]):
                for w in self.tr[u]:
                    scanned += 1
                    wl = w - self.lo
                    if not self.vis[wl]:
                        self.vis[wl] = nxt[wl] = True
                        self.parent[wl] = u
        else:
            for wl in np.flatnonzero(~self.vis):
                v = self.lo + wl
                for u in g.dst[g.row_starts[v] : g.row_starts[v + 1]][::-1]:
                    scanned += 1
                    if bits[u]:
                        self.parent[wl] = u
                        nxt[wl] = True
                        break
            self.vis |= nxt
        found = np.flatnonzero(nxt)
        d = g.degrees[self.lo + found].astype(np.int64)
        deg_next, maxdeg = int(d.sum()), int(d.max()) if d.size else 0
        words = np.zeros(self.n_words_local * 32, bool)
        words[: self.n_local] = nxt
        packed = np.packbits(words, bitorder="little").view(np.int32)
        return np.array([found.size, deg_next, maxdeg, scanned], np.int64), torch.from_numpy(packed.copy())


def _worker(rank, world, port, scale, align, roots, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, e = oracle.kronecker_generate(scale, 8, seed=3)
    g0 = oracle.build_csr(n, e)
    perm, n_plus, _ = oracle.rcm(g0)
    g = oracle.apply_permutation(g0, perm)
    bounds = partition_bounds(g.row_starts, n_plus, world, align)
    local = CpuLocalLevel(g, bounds, rank)
    drv = PartitionedBfs(local, bounds, rank, world, n_policy=g.n, m_directed=g.m_directed)
    out = []
    for s in roots:
        recs = drv.run(int(s), int(g.degrees[s]))
        sizes = [bounds[r + 1] - bounds[r] for r in range(world)]
        par = torch.full((max(sizes),), -1, dtype=torch.int64)
        par[: local.n_local] = torch.from_numpy(local.parent)
        gathered = [torch.zeros(max(sizes), dtype=torch.int64) for _ in sizes]
        dist.all_gather(gathered, par)
        full = torch.cat([gathered[r][: sizes[r]] for r in range(world)])
        out.append(([(r.direction, r.n_f, r.m_f, r.m_u) for r in recs], full.numpy()))
    if rank == 0:
        q.put((bounds, out))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_bfs_gloo_matches_oracle(world):
    scale, align = 11, 256
    n, e = oracle.kronecker_generate(scale, 8, seed=3)
    g0 = oracle.build_csr(n, e)
    perm, n_plus, _ = oracle.rcm(g0)
    g = oracle.apply_permutation(g0, perm)
    roots = oracle.sample_sources(g.degrees, 4, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scale, align, roots, q)) for r in range(world)]
    for p in procs:
        p.start()
    bounds, out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(set(bounds)) > 2  # the graph really is split
    labels = oracle.csr_components(g)
    for s, (recs, par_dev) in zip(roots, out):
        _, rec, _ = oracle.hybrid_bfs(g, int(s))
        want = [tuple(int(x) for x in row[1:5]) for row in rec]
        assert recs == want
        parent = np.full(g.n, -1, np.int32)
        parent[: par_dev.size] = par_dev
        ok, flags, lev = oracle.validate(g, labels, int(s), parent)
        assert ok, flags
        _, want_lev, _, _ = oracle.seq_bfs(g, int(s))
        assert np.array_equal(lev.astype(np.int32), want_lev)
