"""configs[3] path at small scale (GPU): the sharded preprocessing
(paper_2012_10026_b200/sharded.py -- per-rank generation, local build, owner
all-to-all, RCM on the root, all-to-all relabel) over world 2 and 3, as
separate processes sharing the GPU with gloo (host-staged collectives; no
kernel waits on another rank), against the single-GPU pipeline's oracle:
the RCM permutation, every rank's block of the relabelled CSR, and then the
1D-partitioned traversal of that sharded graph (host-driven levels) --
records and trees."""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, scale, q):
    import torch
    import torch.distributed as dist

    import paper_2012_10026_b200 as rb
    from paper_2012_10026_b200.distributed import GpuLocalLevel, PartitionedBfs
    from paper_2012_10026_b200.sharded import build_sharded_rcm_graph, sharded_kronecker_csr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = rb.KroneckerParams(scale=scale, seed=1)
    old = sharded_kronecker_csr(params, rank, world)
    old_rows = (old.lo, old.hi, old.rs.cpu().numpy(), old.col.cpu().numpy())
    rows, bounds, stats, md, perm = build_sharded_rcm_graph(params, rank, world)
    out = {"old": old_rows, "bounds": bounds, "rs": rows.rs.cpu().numpy(), "col": rows.col.cpu().numpy(),
           "perm": perm, "n_plus": stats.n_non_isolated, "md": md, "records": []}
    local = GpuLocalLevel((params.n, md), bounds, rank, 64, 8, True, True, rows=rows)
    drv = PartitionedBfs(local, bounds, rank, world, n_policy=params.n, m_directed=md)
    deg = dist_deg = None
    for s in (3, 17, 123):
        # deg(source): owner rank holds it; all_reduce the (only nonzero) contribution
        lo, hi = bounds[rank], bounds[rank + 1]
        d = torch.tensor([int(rows.deg[s - lo]) if lo <= s < hi else 0], dtype=torch.int64)
        dist.all_reduce(d)
        recs = drv.run(s, int(d.item()))
        out["records"].append((s, [(r.direction, r.n_f, r.m_f, r.m_u) for r in recs],
                               local.parents().cpu().numpy(), local.levels().cpu().numpy()))
    q.put((rank, out))
    dist.barrier()
    local.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("scale,world", [(14, 2), (16, 3)])
def test_sharded_pipeline_matches_single_gpu_oracle(cuda_ok, scale, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, scale, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, e = oracle.kronecker_generate(scale, 16, seed=1)
    g = oracle.build_csr(n, e)
    # step 2: every rank's old-id block == the oracle CSR's rows
    for r in range(world):
        lo, hi, rs, col = res[r]["old"]
        assert np.array_equal(rs, g.row_starts[lo: hi + 1] - g.row_starts[lo]), r
        assert np.array_equal(col.view(np.uint32), g.dst[g.row_starts[lo]: g.row_starts[hi]]), r
    # step 3: the RCM permutation
    perm, n_plus, _ = oracle.rcm(g)
    assert np.array_equal(res[0]["perm"], perm)
    assert res[0]["n_plus"] == n_plus and res[0]["md"] == g.m_directed
    # step 4: every rank's block of the relabelled CSR
    g2 = oracle.apply_permutation(g, perm)
    bounds = res[0]["bounds"]
    assert bounds[0] == 0 and bounds[-1] == n_plus
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        assert np.array_equal(res[r]["rs"], g2.row_starts[lo: hi + 1] - g2.row_starts[lo]), r
        assert np.array_equal(res[r]["col"].view(np.uint32), g2.dst[g2.row_starts[lo]: g2.row_starts[hi]]), r
    # the partitioned traversal of the sharded graph
    labels = oracle.csr_components(g2)
    for i, (s, recs, _, _) in enumerate(res[0]["records"]):
        _, lev, rec, _ = oracle.bfs_run(g2, s, "hybrid", want_levels=True)
        assert recs == [tuple(int(x) for x in row[1:5]) for row in rec], s
        parent = np.full(g2.n, -1, np.int32)
        level = np.full(g2.n, -1, np.int32)
        for r in range(world):
            lo, hi = bounds[r], bounds[r + 1]
            parent[lo:hi] = res[r]["records"][i][2]
            level[lo:hi] = res[r]["records"][i][3]
        ok, flags, _ = oracle.validate(g2, labels, s, parent)
        assert ok, flags
        assert np.array_equal(level, lev)
