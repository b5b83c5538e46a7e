"""Pin the oracle's newer restatements (CPU only):

* C + OpenMP Kronecker / Chung-Lu generators == the numpy restatements
  (generator.py:114-148 with numpy's own Philox) == the reference hashes;
* every BfsEngine mode's full LevelRecords -- scanned, pass1_hits,
  live_vertices, claimed included -- == the reference's (tests/golden/
  modes.json, produced by running rcmbfs for 1 / 3 / 4 threads and partition
  factors 20 / 10 / 1: engine.py:478-604, _kernels.py:90-293, partition.py);
* partial_rcm (reorder.py:240-251), get_partitions / shrink_bounds
  (partition.py:67-171) == reference fixtures (tests/golden/partial.json);
* the product's host-side PartitionSet / Bitmap match the same fixtures.
"""

import warnings

import numpy as np
import pytest

import oracle
import paper_2012_10026_b200 as rb
from conftest import mode_records, sha


@pytest.mark.parametrize("scale,ef,seed", [(6, 4, 3), (10, 16, 42), (13, 16, 5), (16, 16, 7)])
def test_c_kronecker_matches_numpy_and_reference(golden_gen, scale, ef, seed):
    n, e = oracle.kronecker_generate(scale, ef, seed=seed)
    _, e2 = oracle.kronecker_generate_numpy(scale, ef, seed=seed)
    assert np.array_equal(e, e2)
    assert sha(e) == golden_gen[f"{scale},{ef},{seed}"]["edges_sha256"]


@pytest.mark.parametrize("n", [5, 1000, 70000])
def test_c_chunglu_matches_numpy(n):
    _, a = oracle.chunglu_generate(n, seed=7)
    _, b = oracle.chunglu_generate_numpy(n, seed=7)
    assert np.array_equal(a, b)


def test_mode_records_match_reference(golden_modes, ocache):
    for key, cases in golden_modes.items():
        scale, seed = map(int, key.split(","))
        g2 = ocache.kron(scale, seed)["g2"]
        gd = oracle.degree_sort_rows(g2, True)
        labels = oracle.csr_components(g2)
        for c in cases:
            par, lev, rec, _ = oracle.bfs_run(g2, c["source"], c["mode"], threads=c["threads"],
                                              partition_factor=c["partition_factor"], g_desc_dst=gd,
                                              want_levels=True)
            assert mode_records(rec, True) == c["records"], (key, c["mode"], c["threads"], c["source"])
            ok, _, dl = oracle.validate(g2, labels, c["source"], par)
            assert ok and np.array_equal(dl.astype(np.int32), lev)


def test_partial_rcm_matches_reference(golden_partial, ocache):
    for c in golden_partial["partial"]:
        g = ocache.kron(c["scale"], c["seed"])["g"]
        perm, n_plus, ranges = oracle.partial_rcm(g, c["p"])
        assert sha(perm) == c["perm_sha256"], c["p"]
        assert [list(r) for r in ranges] == c["ranges"], c["p"]
        assert min(int(np.ceil(c["p"] * n_plus)), n_plus) == c["n_assigned"]


def test_partitions_and_shrink_match_reference(golden_partial):
    for c in golden_partial["partitions"]:
        st, en = oracle.get_partitions(c["n"], c["factor"], c["threads"])
        assert st.tolist() == c["starts"] and en.tolist() == c["ends"]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ps = rb.get_partitions(c["n"], c["factor"], c["threads"])
        assert ps.starts.tolist() == c["starts"] and ps.ends.tolist() == c["ends"]
        assert ps.live_total() == c["n"] and int(ps.block_counts.sum()) == -(-c["n"] // 512)
    checked = 0
    for c in golden_partial["shrink"]:
        if c["words"] is None:
            continue
        words = np.array(c["words"], np.uint64)
        vis = rb.Bitmap(c["n"])
        vis.words[:] = words
        ps = rb.PartitionSet(n=c["n"], starts=np.array(c["starts"]), ends=np.array(c["ends"]),
                             live_lo=np.array(c["starts"]), live_hi=np.array(c["ends"]), cursor=np.zeros(1, np.int64))
        for i, want in enumerate(c["result"]):
            assert list(rb.shrink_partition(ps, i, vis)) == want
            assert list(oracle.shrink_bounds(words, words, c["starts"][i], c["ends"][i])) == want
        checked += 1
    assert checked >= 10


def test_partition_api_errors():
    with pytest.raises(ValueError, match="at least one vertex"):
        rb.get_partitions(0, 1, 1)
    with pytest.raises(ValueError, match="must be >= 1"):
        rb.get_partitions(10, 0, 1)
    with pytest.warns(UserWarning, match="clamped from 20 to 1"):
        ps = rb.get_partitions(100, 20, 1)
    with pytest.raises(IndexError, match="partition 1 out of range for 1"):
        rb.shrink_partition(ps, 1, rb.Bitmap(100))
    with pytest.raises(ValueError, match="bitmap covers 99 bits"):
        rb.shrink_partition(ps, 0, rb.Bitmap(99))


def test_bitmap_api_matches_reference_semantics():
    rng = np.random.default_rng(3)
    for n in (0, 1, 31, 33, 511, 512, 513, 4097, 100003):
        ids = rng.integers(0, max(n, 1), size=n // 3) if n else np.zeros(0, np.int64)
        bm = rb.Bitmap.from_indices(n, ids)
        ref = np.zeros(-(-n // 512) * 8, np.uint64)
        if ids.size:
            np.bitwise_or.at(ref, ids >> 6, np.uint64(1) << (ids & 63).astype(np.uint64))
        assert np.array_equal(bm.words, ref) and (n == 0 or bm.words.ctypes.data % 64 == 0)
        assert bm.count() == len(set(ids.tolist()))
        assert bm.to_indices().tolist() == sorted(set(ids.tolist())) and bm.to_indices().dtype == np.uint32
        c = bm.copy()
        c.clear_all()
        assert c.count() == 0 and bm.count() == len(set(ids.tolist()))
    bm = rb.Bitmap(70)
    assert bm.test_and_set(69) is False and bm.test_and_set(69) is True and bm.test(69)
    with pytest.raises(IndexError, match="bit 70 out of range for bitmap of 70 bits"):
        bm.set(70)
    with pytest.raises(IndexError, match="bit -1 out of range"):
        bm.set_many([3, -1])
    with pytest.raises(ValueError, match="non-negative"):
        rb.Bitmap(-1)
    a, b = rb.Bitmap.from_indices(2000, [1, 600]), rb.Bitmap.from_indices(2000, [2, 1500])
    rb.or_blocks(a, b, 0, 2)
    assert a.to_indices().tolist() == [1, 2, 600]
    rb.copy_blocks(a, b, 2, 4)
    assert a.to_indices().tolist() == [1, 2, 600, 1500]
    with pytest.raises(IndexError, match=r"block range \[0, 5\) invalid for 4 blocks"):
        rb.or_blocks(a, b, 0, 5)
    with pytest.raises(ValueError, match="size mismatch"):
        rb.copy_blocks(a, rb.Bitmap(10), 0, 1)
