"""Device BFS parity (GPU): levels bit-exact with the reference, every parent
tree valid, per-level direction / n_f / m_f / m_u identical.

Graphs here are built by the (pinned) oracle and uploaded, so these tests
isolate the traversal kernels; tests/test_gpu_prep.py covers the device
preprocessing and the full pipeline."""

import warnings

import numpy as np
import pytest

import oracle
import paper_2012_10026_b200 as rb
from conftest import sha, small_graph

pytestmark = pytest.mark.gpu


def to_rb(g):
    return rb.CsrGraph(g.n, g.row_starts, g.dst, g.degrees)


def desc_of(g):
    return rb.CsrGraph(g.n, g.row_starts, oracle.degree_sort_rows(g, True), g.degrees)


def check_run(g_or, labels, res, source, want_levels=None, want_records=None, eng=None):
    ok, flags, lev = oracle.validate(g_or, labels, source, res.predecessor)
    assert ok, (source, flags.tolist())
    if want_levels is not None:
        assert np.array_equal(lev, want_levels)
    if eng is not None and eng.n_dev:
        dl = eng.level_device().cpu().numpy()
        full = np.full(g_or.n, -1, np.int64)
        full[: dl.size] = dl
        assert np.array_equal(full, lev), "device level array != derived levels"
    if want_records is not None:
        got = [["T" if r.direction == rb.TOP_DOWN else "B", r.n_f, r.m_f, r.m_u] for r in res.levels]
        assert got == want_records
    return lev


@pytest.mark.parametrize("key", ["12,1", "14,3", "16,1", pytest.param("18,1", marks=pytest.mark.slow),
                                 pytest.param("20,1", marks=pytest.mark.slow)])
def test_levels_and_records_vs_reference(cuda_ok, golden_kron, ocache, key):
    scale, seed = map(int, key.split(","))
    ref = golden_kron[key]
    c = ocache.kron(scale, seed)
    g2 = c["g2"]
    labels = oracle.csr_components(g2)
    g = to_rb(g2)
    with rb.BfsEngine(g, rb.BfsParams(mode="hybrid"), record_levels=True) as eng:
        assert eng.n_dev == c["n_plus"]  # isolated tail dropped
        for r in ref["roots"]:
            res = eng.run(r["source"])
            lev = check_run(g2, labels, res, r["source"], want_records=r["records"], eng=eng)
            assert sha(lev.astype(np.int32)) == r["levels_sha256"]
            assert res.traversed_edges == r["traversed"]
            assert res.n_reached == r["n_reached"]


def test_modes_agree(cuda_ok, ocache):
    c = ocache.kron(14, 3)
    g2 = c["g2"]
    labels = oracle.csr_components(g2)
    g, gd = to_rb(g2), desc_of(g2)
    srcs = oracle.sample_sources(g2.degrees, 8, 7)
    engines = {m: rb.BfsEngine(g, rb.BfsParams(mode=m), g_desc=gd, record_levels=True) for m in rb.MODES}
    try:
        for s in srcs:
            s = int(s)
            _, want, _, _ = oracle.seq_bfs(g2, s)
            nf_seq = None
            for m, eng in engines.items():
                res = eng.run(s)
                lev = check_run(g2, labels, res, s, eng=eng)
                assert np.array_equal(lev.astype(np.int32), want), m
                nfs = [r.n_f for r in res.levels]
                nf_seq = nf_seq or nfs
                assert nfs == nf_seq, m
    finally:
        for e in engines.values():
            e.close()


def test_level_sync_runs_top_down_only(cuda_ok, ocache):
    """level_sync / sequential never run a bottom-up level (engine.py use_dir =
    TOP_DOWN when hybrid is off): every record is labelled AND executed
    top-down, and a top-down level scans exactly its frontier edges."""
    for scale, seed in ((14, 3), (16, 1)):
        g2 = ocache.kron(scale, seed)["g2"]
        g = to_rb(g2)
        for mode in ("level_sync", "sequential"):
            with rb.BfsEngine(g, rb.BfsParams(mode=mode)) as eng:
                for s in oracle.sample_sources(g2.degrees, 6, scale):
                    res = eng.run(int(s))
                    _, rec, _ = oracle.hybrid_bfs(g2, int(s), hybrid=False)
                    assert [(r.n_f, r.m_f, r.m_u) for r in res.levels] == [tuple(int(x) for x in row[2:5]) for row in rec]
                    for r in res.levels:
                        assert r.direction == rb.TOP_DOWN and r.executed_direction == rb.TOP_DOWN, (mode, s, r)
                        assert r.scanned_edges == r.m_f, (mode, s, r)


def test_direction_patterns_known_answer(cuda_ok, ocache):
    # test_engine.py:406-420
    g2 = ocache.kron(12)["g2"]
    g = to_rb(g2)
    pats = []
    for s in (1401, 2893, 3196, 954):
        res = rb.bfs_run(g, s, rb.BfsParams(mode="hybrid"))
        pats.append("".join("T" if r.direction == rb.TOP_DOWN else "B" for r in res.levels))
    assert pats == ["TBBBT", "TBBBT", "TBBBT", "TTBBT"]


def test_random_graphs_vs_sequential(cuda_ok, golden_small):
    for i in range(len(golden_small["n_list"])):
        n, e = small_graph(golden_small, i)
        g_or = oracle.build_csr(n, e)  # unordered ids: isolated vertices anywhere
        labels = oracle.csr_components(g_or)
        g = to_rb(g_or)
        for mode in ("hybrid", "level_sync"):
            with rb.BfsEngine(g, rb.BfsParams(mode=mode)) as eng:
                for s in list(golden_small[f"g{i}_srcs"]) + [0, n - 1]:
                    s = int(s)
                    _, want, _, _ = oracle.seq_bfs(g_or, s)
                    res = eng.run(s)
                    lev = check_run(g_or, labels, res, s)
                    assert np.array_equal(lev.astype(np.int32), want), (i, mode, s)


def test_alpha_beta_variants_match_oracle_records(cuda_ok, ocache):
    c = ocache.kron(16)
    g2 = c["g2"]
    g = to_rb(g2)
    for alpha, beta in ((1, 1), (14, 24), (128, 32), (64, 2)):
        with rb.BfsEngine(g, rb.BfsParams(alpha=alpha, beta=beta)) as eng:
            for s in oracle.sample_sources(g2.degrees, 4, alpha):
                _, rec, _ = oracle.hybrid_bfs(g2, int(s), alpha=alpha, beta=beta)
                res = eng.run(int(s))
                got = [(0 if r.direction == rb.TOP_DOWN else 1, r.n_f, r.m_f, r.m_u) for r in res.levels]
                assert got == [tuple(int(x) for x in row[1:5]) for row in rec]


def test_edge_cases(cuda_ok):
    # single vertex / isolated source (test_engine.py:127-148, 555-560)
    g = to_rb(oracle.build_csr(1, np.zeros((0, 2), np.uint32)))
    res = rb.bfs_run(g, 0)
    assert list(res.predecessor) == [0] and res.depth == 0 and res.traversed_edges == 0
    g = to_rb(oracle.build_csr(4, np.array([[1, 2]], np.uint32)))
    res = rb.bfs_run(g, 0)
    assert list(res.predecessor) == [0, -1, -1, -1] and res.n_reached == 1
    with pytest.raises(ValueError, match="out of range"):
        rb.bfs_run(g, 4)
    with pytest.raises(ValueError, match="out of range"):
        rb.bfs_run(g, -1)
    # path of 3: (test_engine.py:136-140)
    g = to_rb(oracle.build_csr(3, np.array([[0, 1], [1, 2]], np.uint32)))
    res = rb.bfs_sequential(g, 0)
    assert list(res.predecessor) == [0, 0, 1] and [r.n_f for r in res.levels] == [1, 1, 1]
    with pytest.raises(ValueError, match="descending-degree"):
        rb.BfsEngine(g, rb.BfsParams(mode="hybrid_reduced"))


def test_sequential_parents_equal_reference(cuda_ok, golden_small, ocache):
    """bfs_sequential's predecessor is the reference's first discoverer
    (_kernels.py:26-54): against the reference's own bfs_sequential runs
    (tests/golden/small.npz), and against the pinned oracle on a Kronecker
    graph with ascending and with degree-sorted rows (any row order)."""
    for i in range(len(golden_small["n_list"])):
        n, e = small_graph(golden_small, i)
        g = oracle.build_csr(n, e)
        g2 = oracle.apply_permutation(g, oracle.rcm(g)[0])
        for j, s in enumerate(golden_small[f"g{i}_srcs"]):
            res = rb.bfs_sequential(to_rb(g2), int(s))
            assert np.array_equal(res.predecessor, golden_small[f"g{i}_seqpar_{int(s)}"]), (i, int(s))
    c = ocache.kron(14, 3)
    g2 = c["g2"]
    gd = oracle.Csr(g2.n, g2.row_starts, oracle.degree_sort_rows(g2, True), g2.degrees)
    for g_or in (g2, gd):
        for s in (0, int(np.argmax(g2.degrees)), c["n_plus"] - 1, g2.n - 1):
            want_par, want_lev, _, _ = oracle.seq_bfs(g_or, s)
            res = rb.bfs_sequential(to_rb(g_or), s)
            assert np.array_equal(res.predecessor, want_par), s
            assert [r.direction for r in res.levels] == [rb.TOP_DOWN] * len(res.levels)


def test_deep_path_continues_past_record_cap(cuda_ok):
    k = 9000  # > 4096 levels per launch -> continuation launches
    e = np.stack([np.arange(k - 1), np.arange(1, k)], 1).astype(np.uint32)
    g_or = oracle.build_csr(k, e)
    labels = oracle.csr_components(g_or)
    res = rb.bfs_run(to_rb(g_or), 0, rb.BfsParams(mode="hybrid"))
    assert res.depth == k - 1
    lev = check_run(g_or, labels, res, 0)
    assert np.array_equal(lev, np.arange(k))


def test_hubs_split_across_warps(cuda_ok):
    rng = np.random.default_rng(11)
    # two big stars sharing leaves + a sprinkle of random edges: hub queue + chunking
    n = 20000
    hub_a, hub_b = 0, 1
    la = rng.choice(np.arange(2, n), 9000, replace=False)
    lb = rng.choice(np.arange(2, n), 7000, replace=False)
    extra = rng.integers(2, n, size=(3000, 2))
    e = np.concatenate([np.stack([np.full(la.size, hub_a), la], 1), np.stack([np.full(lb.size, hub_b), lb], 1),
                        extra]).astype(np.uint32)
    g_or = oracle.build_csr(n, e)
    labels = oracle.csr_components(g_or)
    g = to_rb(g_or)
    for mode in ("hybrid", "level_sync"):
        with rb.BfsEngine(g, rb.BfsParams(mode=mode), record_levels=True) as eng:
            for s in (hub_a, hub_b, int(la[0]), int(extra[0, 0])):
                _, want, _, _ = oracle.seq_bfs(g_or, s)
                res = eng.run(s)
                lev = check_run(g_or, labels, res, s, eng=eng)
                assert np.array_equal(lev.astype(np.int32), want)


def test_engine_reuse_is_deterministic_in_levels(cuda_ok, ocache):
    g2 = ocache.kron(14, 3)["g2"]
    g = to_rb(g2)
    with rb.BfsEngine(g, rb.BfsParams()) as eng:
        a = eng.run(5)
        b = eng.run(7)
        c = eng.run(5)
        with pytest.raises(ValueError, match="record_levels"):
            eng.level_device()  # per-vertex levels are opt-in
    la = [r.n_f for r in a.levels]
    assert la == [r.n_f for r in c.levels]
    assert np.array_equal(a.predecessor >= 0, c.predecessor >= 0)
    assert b.source == 7


# ---------------------------------------------------------------------------
# single steps (criterion 2, test_acceptance.py:117-164)


def test_steps_match_reference_fixtures(cuda_ok, golden_small):
    for i in range(len(golden_small["n_list"])):
        n, e = small_graph(golden_small, i)
        g_or = oracle.apply_permutation(oracle.build_csr(n, e), golden_small[f"g{i}_perm"])
        g = to_rb(g_or)
        vis_idx = golden_small[f"g{i}_state_vis"]
        f_idx = golden_small[f"g{i}_state_frontier"]
        for kind, fn in (("td", rb.top_down_step), ("bu", rb.bottom_up_step)):
            visited = rb.Bitmap.from_indices(n, vis_idx)
            parent = np.full(n, -1, np.int32)
            parent[vis_idx] = vis_idx
            fr = rb.Frontier.from_queue(n, f_idx.astype(np.uint32))
            nxt, st = fn(g, fr, visited, parent)
            assert np.array_equal(np.sort(nxt.indices()), golden_small[f"g{i}_{kind}_next"]), (i, kind)
            assert np.array_equal(visited.words, golden_small[f"g{i}_{kind}_visited"]), (i, kind)
            ref_stats = golden_small[f"g{i}_{kind}_stats"]
            assert (st.n_next, st.deg_next) == (int(ref_stats[0]), int(ref_stats[1]))
            if kind == "td":
                assert st.scanned_edges == int(ref_stats[2])
            found = np.sort(nxt.indices()).astype(np.int64)
            fset = set(f_idx.tolist())
            for w in found:  # every discovered vertex adopted a frontier neighbour
                p = int(parent[w])
                assert p in fset and p in g_or.dst[g_or.row_starts[w]:g_or.row_starts[w + 1]]


def test_random_states_all_step_kernels(cuda_ok):
    rng = np.random.default_rng(888)
    states = 0
    for _ in range(12):
        n = int(rng.integers(64, 3000))
        m = max(1, int(n * rng.uniform(1.0, 4.0)))
        g_or = oracle.build_csr(n, rng.integers(0, n, size=(m, 2), dtype=np.uint32))
        g, gd = to_rb(g_or), desc_of(g_or)
        for _ in range(8):
            vis_mask = rng.random(n) < rng.choice([0.15, 0.4, 0.7])
            vis_mask[int(rng.integers(n))] = True
            vis_idx = np.flatnonzero(vis_mask)
            f_idx = vis_idx[rng.random(vis_idx.size) < 0.5]
            if f_idx.size == 0:
                f_idx = vis_idx[:1]
            nw = ((n + 511) // 512) * 8
            ref_vis = np.zeros(nw, np.uint64)
            np.bitwise_or.at(ref_vis, vis_idx >> 6, np.uint64(1) << (vis_idx & 63).astype(np.uint64))
            ref_par = np.full(n, -1, np.int32)
            ref_par[vis_idx] = vis_idx
            nq, _ = oracle.td_step(g_or, f_idx.astype(np.uint32), ref_vis, ref_par)
            want = np.sort(nq)
            for fn, graph in ((rb.top_down_step, g), (rb.top_down_step_balanced, g), (rb.bottom_up_step, g),
                              (rb.bottom_up_step_balanced, g), (rb.bottom_up_step_reduced, gd)):
                visited = rb.Bitmap.from_indices(n, vis_idx)
                parent = np.full(n, -1, np.int32)
                parent[vis_idx] = vis_idx
                nxt, _ = fn(graph, rb.Frontier.from_queue(n, f_idx.astype(np.uint32)), visited, parent)
                assert np.array_equal(np.sort(nxt.indices()), want), fn.__name__
                assert np.array_equal(visited.words, ref_vis), fn.__name__
            states += 1
    assert states == 96


@pytest.mark.parametrize("knobs", [{"RB_DEFER_MF": "0"}, {"RB_DEFER_MF": "0", "RB_SOLO": "0"},
                                   {"RB_EXEC_OPT": "0"}, {"RB_DEFER_MF": "4096", "RB_PROBE_MF": "0"},
                                   {"RB_KB": "8"}, {"RB_KB": "8", "RB_BU_SPARSE": "0"},
                                   {"RB_KB": "8", "RB_EXEC_ALPHA": "1"}])
def test_engine_knobs_keep_parity(cuda_ok, ocache, monkeypatch, knobs):
    """Execution knobs change HOW a level runs (deferred fire-and-forget claims
    counted from the next-frontier bitmap, solo levels, the executed direction,
    probing, the large-graph build with 8-word bottom-up steps and the sparse
    list levels) -- never the levels, the records or tree validity."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    for scale, seed in ((14, 3), (16, 1)):
        c = ocache.kron(scale, seed)
        g2 = c["g2"]
        labels = oracle.csr_components(g2)
        with rb.BfsEngine(to_rb(g2), rb.BfsParams(mode="hybrid"), record_levels=True) as eng:
            for s in oracle.sample_sources(g2.degrees, 6, scale):
                s = int(s)
                _, want, _, _ = oracle.seq_bfs(g2, s)
                _, rec, _ = oracle.hybrid_bfs(g2, s)
                res = eng.run(s)
                lev = check_run(g2, labels, res, s, eng=eng)
                assert np.array_equal(lev.astype(np.int32), want), (knobs, scale, s)
                got = [(0 if r.direction == rb.TOP_DOWN else 1, r.n_f, r.m_f, r.m_u) for r in res.levels]
                assert got == [tuple(int(x) for x in r[1:5]) for r in rec], (knobs, scale, s)


# ---------------------------------------------------------------------------
# the paper's partitioned modes: every LevelRecord field vs the reference


def test_partitioned_modes_match_reference_records(cuda_ok, golden_modes, ocache):
    from conftest import mode_records

    for key, cases in golden_modes.items():
        scale, seed = map(int, key.split(","))
        g2 = ocache.kron(scale, seed)["g2"]
        labels = oracle.csr_components(g2)
        g, gd = to_rb(g2), desc_of(g2)
        engines = {}
        try:
            for c in cases:
                k = (c["mode"], c["threads"], c["partition_factor"])
                if k not in engines:
                    with warnings.catch_warnings():
                        warnings.simplefilter("ignore")
                        engines[k] = rb.BfsEngine(g, rb.BfsParams(mode=c["mode"], threads=c["threads"],
                                                                  partition_factor=c["partition_factor"]),
                                                  g_desc=gd)
                res = engines[k].run(c["source"])
                assert mode_records(res.levels, False) == c["records"], (key, k, c["source"])
                check_run(g2, labels, res, c["source"])
        finally:
            for e in engines.values():
                e.close()


def test_reduced_mode_records_vs_oracle_random_graphs(cuda_ok):
    """live_vertices edge cases: isolated vertices inside the range and in
    the tail, n not a multiple of 512, single-block partitions."""
    from conftest import mode_records

    rng = np.random.default_rng(77)
    for it in range(16):
        n = int(rng.integers(300, 9000))
        m = int(n * rng.uniform(0.4, 3.0))
        e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
        g_or = oracle.build_csr(n, e)
        if it % 2:  # RCM graph: isolated tail dropped on device
            g_or = oracle.apply_permutation(g_or, oracle.rcm(g_or)[0])
        gd = oracle.degree_sort_rows(g_or, True)
        labels = oracle.csr_components(g_or)
        threads, lam = int(rng.integers(1, 5)), int(rng.integers(1, 12))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            eng = rb.BfsEngine(to_rb(g_or), rb.BfsParams(mode="hybrid_reduced", threads=threads, partition_factor=lam),
                               g_desc=rb.CsrGraph(n, g_or.row_starts, gd, g_or.degrees))
        with eng:
            for s in rng.choice(np.flatnonzero(g_or.degrees > 0), size=4, replace=False):
                _, _, rec, _ = oracle.bfs_run(g_or, int(s), "hybrid_reduced", threads=threads, partition_factor=lam,
                                              g_desc_dst=gd)
                res = eng.run(int(s))
                assert mode_records(res.levels, False) == mode_records(rec, True), (it, int(s))
                check_run(g_or, labels, res, int(s))
