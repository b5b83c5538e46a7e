"""Chung-Lu generator (BASELINE configs[4]) on device: byte-identical with the
numpy restatement of the recipe, and the full RCM + BFS pipeline on it is
bit-exact with the oracle (hub-heavy graph: exercises hub splitting)."""

import numpy as np
import pytest

import oracle
import paper_2012_10026_b200 as rb
from conftest import sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,avg,gamma,cap,seed", [(1 << 16, 20, 2.1, 0.01, 7), (100003, 7, 2.5, 0.05, 123),
                                                  (5, 4, 2.1, 1.0, 1)])
def test_device_generator_matches_recipe(cuda_ok, n, avg, gamma, cap, seed):
    p = rb.ChungLuParams(n=n, avg_degree=avg, gamma=gamma, cap_frac=cap, seed=seed)
    got = rb.chunglu_generate(p)
    _, want = oracle.chunglu_generate(n, avg, gamma, 1.0, cap, seed)
    assert got.edges.shape == want.shape
    assert np.array_equal(got.edges, want)
    d = rb.chunglu_generate(p, device=True)
    assert sha(d.edges.cpu().numpy().view(np.uint32)) == sha(want)


def test_chunglu_pipeline_bit_exact(cuda_ok):
    n, e = oracle.chunglu_generate(1 << 16)
    go = oracle.build_csr(n, e)
    perm, k, ranges = oracle.rcm(go)
    g2o = oracle.apply_permutation(go, perm)
    el = rb.chunglu_generate(rb.ChungLuParams(n=1 << 16))
    g = rb.build_csr(el)
    assert np.array_equal(g.row_starts, go.row_starts) and np.array_equal(g.dst, go.dst)
    p, st = rb.rcm(g)
    assert np.array_equal(p.perm, perm) and st.component_ranges == ranges
    g2 = rb.apply_permutation(g, p)
    assert np.array_equal(g2.dst, g2o.dst)
    labels = oracle.csr_components(g2o)
    v = rb.Validator(g2)
    with rb.BfsEngine(g2, rb.BfsParams(), record_levels=True) as eng:
        for s in rb.sample_sources(g2.degrees, 16, 1):
            s = int(s)
            res = eng.run(s)
            ok, flags, lev = oracle.validate(g2o, labels, s, res.predecessor)
            assert ok, flags
            _, want, _, _ = oracle.seq_bfs(g2o, s)
            assert np.array_equal(lev.astype(np.int32), want)
            _, rec, _ = oracle.hybrid_bfs(g2o, s)
            assert [(0 if r.direction == rb.TOP_DOWN else 1, r.n_f, r.m_f, r.m_u) for r in res.levels] == \
                [tuple(int(x) for x in row[1:5]) for row in rec]
            assert v.validate(s, res.predecessor).passed
