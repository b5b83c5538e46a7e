"""The 1D partition with the exchange on the device (rb_bfs.cu
bfs_dist / bfs_dist_emu): one persistent launch per root, next-frontier
words and counters stored straight into every rank's buffers.

One GPU, as the profiling guide prescribes for fewer GPUs than ranks: world 2
and 3 as ONE cooperative launch over all ranks' data (the publish, the
triple-buffered global bitmaps and the counter slots exactly as on several
GPUs; the cross-rank barrier becomes a grid barrier); and the real
multi-process path at world 1 (IPC handles, system-scope barrier, loopback).
Checked against the oracle: level records (direction, n_f, m_f, m_u), the
level array, and every parent tree through the five validator rules."""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _graph(kind, scale):
    import paper_2012_10026_b200 as rb

    if kind == "kron":
        el = rb.kronecker_generate(rb.KroneckerParams(scale=scale, seed=1), device=True)
    else:
        el = rb.chunglu_generate(rb.ChungLuParams(n=1 << scale, seed=7), device=True)
    g = rb.build_csr(el)
    perm, st = rb.rcm(g)
    return rb.apply_permutation(g, perm), st.n_non_isolated


def _check_against_oracle(g2, n_plus, bounds, roots, runs):
    go = oracle.Csr(g2.n, g2.row_starts, g2.dst, g2.degrees)
    labels = oracle.csr_components(go)
    for s, (recs, parent_parts, level_parts) in zip(roots, runs):
        _, lev_or, rec_or, _ = oracle.bfs_run(go, int(s), "hybrid", want_levels=True)
        assert [(r.direction, r.n_f, r.m_f, r.m_u) for r in recs] == \
            [tuple(int(x) for x in row[1:5]) for row in rec_or], int(s)
        parent = np.full(g2.n, -1, np.int32)
        level = np.full(g2.n, -1, np.int32)
        for r in range(len(bounds) - 1):
            parent[bounds[r]:bounds[r + 1]] = parent_parts[r]
            level[bounds[r]:bounds[r + 1]] = level_parts[r]
        ok, flags, _ = oracle.validate(go, labels, int(s), parent)
        assert ok, (int(s), flags.tolist())
        assert np.array_equal(level, lev_or), int(s)


@pytest.mark.parametrize("kind,scale,world", [("kron", 16, 2), ("kron", 16, 3), ("chunglu", 15, 2),
                                              ("kron", 18, 3)])
def test_emulated_ranks_match_oracle(cuda_ok, kind, scale, world):
    import paper_2012_10026_b200 as rb
    from paper_2012_10026_b200.distributed import DevicePartition, connect_emulated, partition_bounds, run_emulated

    g2, n_plus = _graph(kind, scale)
    bounds = partition_bounds(g2.row_starts, n_plus, world, 128)
    assert all(bounds[r + 1] > bounds[r] for r in range(world)), bounds
    parts = [DevicePartition(g2, bounds, r, world, record_levels=True) for r in range(world)]
    try:
        connect_emulated(parts)
        deg = g2.degrees
        roots = rb.sample_sources(deg, 8, 5)
        runs = []
        for s in roots:
            recs, executed, secs = run_emulated(parts, int(s), int(deg[s]))
            assert secs > 0 and len(executed) == len(recs)
            runs.append((recs, [p.local.parents().cpu().numpy() for p in parts],
                         [p.local.levels().cpu().numpy() for p in parts]))
        _check_against_oracle(g2, n_plus, bounds, roots, runs)
    finally:
        for p in parts:
            p.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_multiprocess_path_world1_loopback(cuda_ok):
    """The real multi-GPU path (IPC handle exchange, peer stores, system-scope
    cross-rank barrier carried across roots) with one rank: its peer is itself."""
    import torch
    import torch.distributed as dist

    import paper_2012_10026_b200 as rb
    from paper_2012_10026_b200.distributed import DeviceExchangeBfs, partition_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        g2, n_plus = _graph("kron", 16)
        bounds = partition_bounds(g2.row_starts, n_plus, 1, 128)
        drv = DeviceExchangeBfs(g2, bounds, 0, 1, record_levels=True)
        roots = rb.sample_sources(g2.degrees, 6, 9)
        runs = []
        for s in roots:
            recs = drv.run(int(s), int(g2.degrees[s]))
            runs.append((recs, [drv.local.parents().cpu().numpy()], [drv.local.levels().cpu().numpy()]))
            assert drv.elapsed() > 0
        _check_against_oracle(g2, n_plus, bounds, roots, runs)
        drv.close()
    finally:
        dist.destroy_process_group()
