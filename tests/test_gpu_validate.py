"""GPU tree validator (csrc/rb_validate.cu) vs the pinned oracle validator and
the reference's fault-injection cases (test_validate.py:23-178): each rule is
isolated by a targeted fault, the report texts match, derived levels match."""

import numpy as np
import pytest

import oracle
import paper_2012_10026_b200 as rb

pytestmark = pytest.mark.gpu

NAMES = ["source is own parent", "tree edges exist", "parent chains are proper levels",
         "edges span at most one level", "reachability matches components"]


def vec(rep):
    assert [c.name for c in rep.checks] == NAMES
    return [c.passed for c in rep.checks]


def to_rb(go):
    return rb.CsrGraph(go.n, go.row_starts, go.dst, go.degrees)


@pytest.fixture(scope="module")
def base(cuda_ok):
    # Kronecker scale 10 (reference conftest kron.graph(10)): edgefactor 16, seed 1
    n, e = oracle.kronecker_generate(10)
    go = oracle.build_csr(n, e)
    g = to_rb(go)
    v = rb.Validator(g)
    source = int(np.argmax(go.degrees))
    parent, levels, _, _ = oracle.seq_bfs(go, source)
    parent = parent.astype(np.int32)
    return go, g, v, source, parent, levels.astype(np.int64)


def test_valid_trees_and_levels(base):
    go, g, v, source, parent, levels = base
    rep = v.validate(source, parent)
    assert rep.passed and vec(rep) == [True] * 5
    assert np.array_equal(rep.derived_levels, levels)
    assert rep.as_text().splitlines()[0] == "validation: PASS"
    kv = rep.as_key_values()
    assert "passed = true" in kv and "check.tree_edges_exist = true" in kv


def test_fault_source_not_own_parent(base):
    go, g, v, source, parent, _ = base
    bad = parent.copy()
    bad[source] = go.dst[go.row_starts[source]]
    rep = v.validate(source, bad)
    assert vec(rep) == [False, True, True, True, True]
    txt = rep.as_text()
    assert "[FAIL] source is own parent" in txt and f"parent[{source}]" in txt
    assert "check.source_is_own_parent.detail" in rep.as_key_values()


def test_fault_phantom_tree_edge(base):
    go, g, v, source, parent, levels = base
    bad = parent.copy()
    done = False
    for lv in range(2, int(levels.max()) + 1):
        above = np.flatnonzero(levels == lv - 1)
        for x in np.flatnonzero(levels == lv):
            nb = set(go.dst[go.row_starts[x] : go.row_starts[x + 1]].tolist())
            cand = [u for u in above if int(u) not in nb]
            if cand:
                bad[x] = cand[0]
                done = True
                break
        if done:
            break
    assert done
    rep = v.validate(source, bad)
    assert vec(rep) == [True, False, True, True, True]
    assert "is not a graph edge" in rep.checks[1].detail


def test_fault_parent_cycle(base):
    go, g, v, source, parent, _ = base
    bad = parent.copy()

    def nbrs(x):
        return go.dst[go.row_starts[x] : go.row_starts[x + 1]]

    a = next(x for x in range(go.n) if x != source and parent[x] >= 0
             and any(int(w) != source and parent[w] >= 0 for w in nbrs(x)))
    b = next(int(w) for w in nbrs(a) if int(w) != source and parent[w] >= 0)
    bad[a], bad[b] = b, a
    rep = v.validate(source, bad)
    ok, flags, _ = oracle.validate(go, oracle.csr_components(go), source, bad)
    assert vec(rep) == flags.tolist()
    assert vec(rep)[2] is False and "never reaches the source" in rep.checks[2].detail


def test_fault_edge_spanning_levels(base):
    go, g, v, source, parent, levels = base
    reach = np.flatnonzero(parent >= 0)
    has_child = np.zeros(go.n, bool)
    has_child[parent[reach]] = True
    bad = parent.copy()
    done = False
    for x in reach:
        x = int(x)
        if x == source or has_child[x]:
            continue
        deeper = [int(u) for u in go.dst[go.row_starts[x] : go.row_starts[x + 1]] if levels[u] == levels[x] + 1]
        if deeper:
            bad[x] = deeper[0]
            done = True
            break
    assert done
    rep = v.validate(source, bad)
    assert vec(rep) == [True, True, True, False, True]
    assert "spans levels" in rep.checks[3].detail


def test_fault_dropped_and_foreign_vertex(base):
    go, g, v, source, parent, _ = base
    reach = np.flatnonzero(parent >= 0)
    has_child = np.zeros(go.n, bool)
    has_child[parent[reach]] = True
    x = next(int(y) for y in reach if int(y) != source and not has_child[int(y)])
    bad = parent.copy()
    bad[x] = -1
    rep = v.validate(source, bad)
    assert vec(rep) == [True, True, True, True, False]
    assert "component but unreached" in rep.checks[4].detail
    iso = np.flatnonzero(go.degrees == 0)
    assert iso.size
    w = int(iso[0])
    bad = parent.copy()
    bad[w] = w
    rep = v.validate(source, bad)
    assert not rep.passed and not rep.checks[4].passed
    assert "outside the source component" in rep.checks[4].detail


def test_component_labels_are_min_ids(cuda_ok):
    e = np.array([[0, 1], [1, 2], [2, 0], [3, 4], [4, 5], [5, 3]], np.uint32)
    el = rb.EdgeList(7, e)
    g = rb.build_csr(el)
    assert rb.Validator(g).component_labels().tolist() == [0, 0, 0, 3, 3, 3, 6]
    assert rb.Validator(g, edge_list=el).component_labels().tolist() == [0, 0, 0, 3, 3, 3, 6]


def test_raw_edge_route_matches_csr_route_and_oracle(cuda_ok):
    el = rb.kronecker_generate(rb.KroneckerParams(scale=12, seed=1))
    g = rb.build_csr(el)
    a = rb.Validator(g, edge_list=el).component_labels()
    b = rb.Validator(g).component_labels()
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle.components(g.n, el.edges))


def test_input_errors(base):
    go, g, v, source, parent, _ = base
    with pytest.raises(ValueError, match="shape"):
        v.validate(source, parent[:-1])
    with pytest.raises(ValueError, match="out of range"):
        v.validate(go.n, parent)


def test_random_graphs_random_faults_vs_oracle(cuda_ok):
    # every rule flag and the derived levels agree with the oracle on random
    # multi-component graphs under random corruptions
    rng = np.random.default_rng(11)
    for _ in range(25):
        n = int(rng.integers(5, 800))
        e = rng.integers(0, n, size=(int(n * rng.choice([0.5, 1.0, 2.5])), 2), dtype=np.uint32)
        go = oracle.build_csr(n, e)
        labels = oracle.csr_components(go)
        v = rb.Validator(to_rb(go))
        src = int(rng.integers(0, n))
        parent = oracle.seq_bfs(go, src)[0].astype(np.int32)
        for trial in range(4):
            bad = parent.copy()
            if trial:
                k = int(rng.integers(1, 4))
                idx = rng.integers(0, n, size=k)
                bad[idx] = rng.integers(-1, n, size=k)
            ok, flags, lev = oracle.validate(go, labels, src, bad)
            rep = v.validate(src, bad)
            assert vec(rep) == flags.tolist(), (n, src, trial)
            assert rep.passed == ok
            assert np.array_equal(rep.derived_levels, lev)


def test_validates_engine_trees_device_side(cuda_ok):
    # the device path: parents stay in HBM, levels equal the oracle's
    el = rb.kronecker_generate(rb.KroneckerParams(scale=16, seed=1))
    g = rb.build_csr(el)
    perm, _ = rb.rcm(g)
    g2 = rb.apply_permutation(g, perm)
    v = rb.Validator(g2)
    g2o = oracle.Csr(g2.n, g2.row_starts, g2.dst, g2.degrees)
    with rb.BfsEngine(g2, rb.BfsParams()) as eng:
        for s in rb.sample_sources(g2.degrees, 4, 1):
            res = eng.run(int(s))
            rep = v.validate(int(s), res.predecessor)
            assert rep.passed, rep.as_text()
            want = oracle.seq_bfs(g2o, int(s))[1]
            assert np.array_equal(rep.derived_levels, want.astype(np.int64))


def test_matches_reference_validator_fixtures(cuda_ok, golden_validate):
    # the reference's own Validator output (check vector, texts, derived levels)
    from conftest import validate_cases

    vals = {}
    for n, e, src, parent, checks, levels, details in validate_cases(golden_validate):
        key = (n, e.tobytes())
        if key not in vals:
            vals[key] = rb.Validator(rb.build_csr(rb.EdgeList(n, e)))
        rep = vals[key].validate(src, parent)
        assert vec(rep) == checks
        assert [c.detail for c in rep.checks] == details
        assert np.array_equal(rep.derived_levels, levels)
