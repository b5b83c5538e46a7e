"""Device preprocessing parity (GPU): build_csr, rcm, apply_permutation and
degree_sort_adjacency are bit-exact with the reference (fixtures from the
reference itself, and the pinned oracle), plus the full pipeline."""

import os

import numpy as np
import pytest

import oracle
import paper_2012_10026_b200 as rb
from conftest import GOLDEN, sha, small_graph

pytestmark = pytest.mark.gpu


def test_device_generator_byte_identical(cuda_ok, golden_gen):
    # generator.py:134-148 restated on device (csrc/rb_gen.cu)
    for key, ref in golden_gen.items():
        scale, ef, seed = map(int, key.split(","))
        el = rb.kronecker_generate(rb.KroneckerParams(scale=scale, edgefactor=ef, seed=seed))
        assert el.edges.dtype == np.uint32 and el.edges.shape == ((1 << scale) * ef, 2)
        assert sha(el.edges) == ref["edges_sha256"], key
    el = rb.kronecker_generate(rb.KroneckerParams(scale=13, edgefactor=16, seed=5), device=True)
    assert sha(el.edges.cpu().numpy().view(np.uint32)) == golden_gen["13,16,5"]["edges_sha256"]
    # other initiators / seeds vs the numpy restatement
    for scale, ef, seed, init in ((9, 3, 123456789, (0.45, 0.15, 0.15, 0.25)), (11, 5, 2**63 + 7, (0.25,) * 4)):
        n, want = oracle.kronecker_generate(scale, ef, init, seed)
        got = rb.kronecker_generate(rb.KroneckerParams(scale=scale, edgefactor=ef, initiator=init, seed=seed))
        assert np.array_equal(got.edges, want)


def test_build_csr_matches_reference_fixtures(cuda_ok, golden_gen):
    for key, ref in golden_gen.items():
        scale, ef, seed = map(int, key.split(","))
        el = rb.kronecker_generate(rb.KroneckerParams(scale=scale, edgefactor=ef, seed=seed))
        g = rb.build_csr(el)
        assert g.m_directed == ref["m_directed"], key
        assert g.isolated_count == ref["isolated"], key
        assert sha(g.row_starts) == ref["row_starts_sha256"], key
        assert sha(g.dst) == ref["dst_sha256"], key


def test_build_csr_known_answers_and_errors(cuda_ok):
    g = rb.build_csr(rb.EdgeList(3, np.array([[0, 1], [1, 0], [1, 1], [0, 1]], np.uint32)))
    assert g.row_starts.tolist() == [0, 1, 2, 2] and g.dst.tolist() == [1, 0] and g.degrees.tolist() == [1, 1, 0]
    with pytest.raises(ValueError, match=r"edge 1 = \(2, 5\) out of range for n=4"):
        rb.build_csr(rb.EdgeList(4, np.array([[0, 1], [2, 5], [9, 9]], np.uint32)))
    g = rb.build_csr(rb.EdgeList(5, np.zeros((0, 2), np.uint32)))
    assert g.m_directed == 0 and g.row_starts.tolist() == [0] * 6
    g = rb.build_csr(rb.EdgeList(3, np.array([[1, 1], [2, 2]], np.uint32)))  # self-loops only
    assert g.m_directed == 0 and g.isolated_count == 3
    with pytest.raises(ValueError, match="non-negative"):
        rb.build_csr(rb.EdgeList(-1, np.zeros((0, 2), np.uint32)))


def test_build_csr_random_vs_oracle(cuda_ok):
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = int(rng.integers(1, 5000))
        m = int(rng.integers(0, 4 * n + 1))
        e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
        want = oracle.build_csr(n, e)
        got = rb.build_csr(rb.EdgeList(n, e))
        assert np.array_equal(got.row_starts, want.row_starts)
        assert np.array_equal(got.dst, want.dst)
        assert np.array_equal(got.degrees, want.degrees)


def test_rcm_small_fixtures(cuda_ok, golden_small):
    for i in range(len(golden_small["n_list"])):
        n, e = small_graph(golden_small, i)
        g = rb.build_csr(rb.EdgeList(n, e))
        perm, st = rb.rcm(g)
        assert np.array_equal(perm.perm, golden_small[f"g{i}_perm"]), i
        inv = np.empty(n, np.uint32)
        inv[perm.perm] = np.arange(n, dtype=np.uint32)
        assert np.array_equal(perm.inv, inv)
        want = golden_small[f"g{i}_ranges"]
        assert np.array_equal(np.array(st.component_ranges, np.int64).reshape(-1, 2), want), i
        assert st.n_non_isolated == n - g.isolated_count and st.complete
        g2 = rb.apply_permutation(g, perm)
        assert np.array_equal(g2.dst, golden_small[f"g{i}_rcm_dst"]), i


def test_rcm_random_multicomponent_vs_oracle(cuda_ok):
    rng = np.random.default_rng(42)
    for _ in range(30):
        n = int(rng.integers(2, 3000))
        m = int(rng.integers(0, int(n * rng.choice([0.2, 0.6, 1.5, 3.0])) + 1))
        e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
        g_or = oracle.build_csr(n, e)
        want_perm, k, want_ranges = oracle.rcm(g_or)
        g = rb.build_csr(rb.EdgeList(n, e))
        perm, st = rb.rcm(g)
        assert np.array_equal(perm.perm, want_perm)
        assert st.component_ranges == want_ranges
        assert st.n_non_isolated == k


@pytest.mark.parametrize("key", ["12,1", "14,3", "16,1", pytest.param("18,1", marks=pytest.mark.slow),
                                 pytest.param("20,1", marks=pytest.mark.slow)])
def test_kron_pipeline_bit_exact(cuda_ok, golden_kron, key):
    scale, seed = map(int, key.split(","))
    ref = golden_kron[key]
    el = rb.kronecker_generate(rb.KroneckerParams(scale=scale, seed=seed))
    g = rb.build_csr(el)
    perm, st = rb.rcm(g)
    assert sha(perm.perm) == ref["perm_sha256"]
    assert st.n_components == ref["n_components"]
    assert sha(np.array(st.component_ranges, np.int64)) == ref["component_ranges_sha256"]
    g2 = rb.apply_permutation(g, perm)
    assert sha(g2.dst) == ref["rcm_dst_sha256"]
    assert sha(g2.row_starts) == ref["rcm_row_starts_sha256"]
    if scale == 12:
        assert np.array_equal(perm.perm, np.load(os.path.join(GOLDEN, "kron12_perm.npy")))
    # BFS on the device-built graph: levels + records vs the reference
    labels = oracle.csr_components(oracle.Csr(g2.n, g2.row_starts, g2.dst, g2.degrees))
    g2o = oracle.Csr(g2.n, g2.row_starts, g2.dst, g2.degrees)
    with rb.BfsEngine(g2, rb.BfsParams()) as eng:
        for r in ref["roots"][:16]:
            res = eng.run(r["source"])
            ok, flags, lev = oracle.validate(g2o, labels, r["source"], res.predecessor)
            assert ok, flags
            assert sha(lev.astype(np.int32)) == r["levels_sha256"]
            assert [["T" if x.direction == rb.TOP_DOWN else "B", x.n_f, x.m_f, x.m_u] for x in res.levels] == r["records"]


def test_degree_sort_adjacency_vs_oracle(cuda_ok):
    rng = np.random.default_rng(9)
    for _ in range(10):
        n = int(rng.integers(2, 3000))
        e = rng.integers(0, n, size=(int(n * 3), 2), dtype=np.uint32)
        g_or = oracle.build_csr(n, e)
        g = rb.build_csr(rb.EdgeList(n, e))
        for order in ("ascending", "descending"):
            got = rb.degree_sort_adjacency(g, order)
            assert np.array_equal(got.dst, oracle.degree_sort_rows(g_or, order == "descending"))
    with pytest.raises(ValueError):
        rb.degree_sort_adjacency(g, "sideways")


def test_apply_permutation_errors_and_identity(cuda_ok):
    g = rb.build_csr(rb.EdgeList(5, np.array([[0, 1], [1, 2], [3, 4]], np.uint32)))
    with pytest.raises(ValueError, match="permutation size 4 != graph size 5"):
        rb.apply_permutation(g, rb.Permutation.identity(4))
    g2 = rb.apply_permutation(g, rb.Permutation.identity(5))
    assert np.array_equal(g2.dst, g.dst)
    with pytest.raises(ValueError, match="bijection"):
        rb.Permutation.from_new_to_orig(np.array([0, 0, 1], np.uint32))


def test_bandwidth_reduction(cuda_ok):
    # criterion 3 (test_acceptance.py:169-184) on device-built graphs
    for scale, seed in [(14, 1), (14, 2), (16, 4)]:
        g = rb.build_csr(rb.kronecker_generate(rb.KroneckerParams(scale=scale, seed=seed)))
        pre = rb.bandwidth(g)
        perm, _ = rb.rcm(g)
        post = rb.bandwidth(rb.apply_permutation(g, perm))
        assert post < g.n - g.isolated_count and post < pre
