"""1D-partition BFS on the GPU: the partitioned kernel path
(owned rows for bottom-up, transpose slice for top-down, global frontier
bitmap from the all-gather) checked against the oracle.  One GPU: world_size 1
over NCCL, and world_size 2 as two processes sharing the GPU with gloo
collectives staged through host memory (host-driven levels: no kernel waits on
another rank)."""

import os
import socket

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(scale, seed):
    import paper_2012_10026_b200 as rb

    el = rb.kronecker_generate(rb.KroneckerParams(scale=scale, seed=seed), device=True)
    g = rb.build_csr(el)
    perm, st = rb.rcm(g)
    return rb.apply_permutation(g, perm), st.n_non_isolated


def _run_ranks(rank, world, backend, port, scale, align, q):
    import torch.distributed as dist

    import paper_2012_10026_b200 as rb
    from paper_2012_10026_b200.distributed import GpuLocalLevel, PartitionedBfs, partition_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    kw = dict(device_id=torch.device("cuda", 0)) if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    g2, n_plus = _graph(scale, 1)
    bounds = partition_bounds(g2.row_starts, n_plus, world, align)
    local = GpuLocalLevel(g2, bounds, rank, alpha=64, beta=8, record_levels=True)
    drv = PartitionedBfs(local, bounds, rank, world, n_policy=g2.n, m_directed=g2.m_directed)
    roots = rb.sample_sources(g2.degrees, 6, 3)
    out = []
    for s in roots:
        recs = drv.run(int(s), int(g2.degrees[s]))
        par = local.parents().cpu().numpy().astype(np.int64) if local.n_local else np.zeros(0, np.int64)
        lev = local.levels().cpu().numpy().astype(np.int64) if local.n_local else np.zeros(0, np.int64)
        out.append((int(s), [(r.direction, r.n_f, r.m_f, r.m_u) for r in recs], par, lev))
    q.put((rank, bounds, out))
    dist.barrier()
    local.close()
    dist.destroy_process_group()


def _check(scale, world, backend, align):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_ranks, args=(r, world, backend, port, scale, align, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, bounds, out = q.get(timeout=600)
        res[rank] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, e = oracle.kronecker_generate(scale, 16, seed=1)
    g0 = oracle.build_csr(n, e)
    perm, n_plus, _ = oracle.rcm(g0)
    g = oracle.apply_permutation(g0, perm)
    labels = oracle.csr_components(g)
    for i in range(len(res[0])):
        s = res[0][i][0]
        _, rec, _ = oracle.hybrid_bfs(g, s)
        assert res[0][i][1] == [tuple(int(x) for x in row[1:5]) for row in rec]
        parent = np.full(g.n, -1, np.int32)
        level = np.full(g.n, -1, np.int64)
        for r in range(world):
            lo, hi = bounds[r], bounds[r + 1]
            parent[lo:hi] = res[r][i][2]
            level[lo:hi] = res[r][i][3]
        ok, flags, lev = oracle.validate(g, labels, s, parent)
        assert ok, flags
        assert np.array_equal(lev, level)
    return bounds


def test_partitioned_world1_nccl(cuda_ok):
    _check(14, 1, "nccl", 8192)


def test_partitioned_world2_one_gpu_gloo(cuda_ok):
    bounds = _check(14, 2, "gloo", 256)
    assert 0 < bounds[1] < bounds[2]
