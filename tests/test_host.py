"""Host-side logic of the drop-in package (no GPU): parameter validation,
direction policy (engine.py:215-228, thresholds from test_engine.py:258-279),
Bitmap layout, Frontier forms, generator byte-identity, and that the C-ABI
library loads and exports every symbol include/rcmbfs_b200.h declares."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2012_10026_b200 as rb
from conftest import ROOT, sha
from paper_2012_10026_b200 import _build, _lib


def policy(direction, m_f, m_u, n_f, n, **kw):
    return rb.update_traversal_policy(
        rb.PolicyCounters(direction=direction, m_f=m_f, m_u=m_u, n_f=n_f, n=n), rb.BfsParams(**kw)
    )


def test_policy_thresholds():
    assert policy(rb.TOP_DOWN, 0, 10_000, 0, 1000) == rb.TOP_DOWN
    assert policy(rb.TOP_DOWN, 101, 6400, 5, 1000) == rb.BOTTOM_UP
    assert policy(rb.TOP_DOWN, 100, 6400, 5, 1000) == rb.TOP_DOWN
    assert policy(rb.BOTTOM_UP, 1, 1, 99, 800) == rb.TOP_DOWN
    assert policy(rb.BOTTOM_UP, 1, 1, 100, 800) == rb.BOTTOM_UP
    assert policy(rb.TOP_DOWN, 11, 100, 5, 1000, alpha=10) == rb.BOTTOM_UP
    assert policy(rb.TOP_DOWN, 11, 100, 5, 1000, alpha=5) == rb.TOP_DOWN
    assert policy(rb.BOTTOM_UP, 1, 1, 400, 1000, beta=2) == rb.TOP_DOWN
    assert policy(rb.BOTTOM_UP, 1, 1, 600, 1000, beta=2) == rb.BOTTOM_UP


def test_params_validation():
    for kw in (dict(alpha=0), dict(alpha=129), dict(beta=0), dict(beta=33), dict(partition_factor=0),
               dict(threads=0), dict(mode="inward")):
        with pytest.raises(ValueError):
            rb.BfsParams(**kw)
    assert rb.default_partition_factor(1 << 25) == 10 and rb.default_partition_factor(1 << 26) == 20


def test_bitmap_layout_and_words32():
    rng = np.random.default_rng(3)
    for n in (1, 31, 32, 63, 64, 511, 512, 513, 4097):
        ids = np.unique(rng.integers(0, n, size=min(n, 50)))
        bm = rb.Bitmap.from_indices(n, ids)
        assert bm.words.ctypes.data % 64 == 0 and bm.n_words == bm.n_blocks * 8
        w32 = bm.words32()
        assert w32.size == (n + 31) // 32
        for i in ids:
            assert (w32[i >> 5] >> (i & 31)) & 1
        back = rb.Bitmap.from_words32(n, np.full(w32.size, 0xFFFFFFFF, np.uint32))
        assert back.count() == n  # padding cleared
        assert np.array_equal(bm.to_indices(), ids.astype(np.uint32))
        assert bm.count() == ids.size


def test_bitmap_scalar_ops():
    bm = rb.Bitmap(100)
    assert not bm.test_and_set(7) and bm.test_and_set(7) and bm.test(7)
    with pytest.raises(IndexError):
        bm.test(100)
    a, b = rb.Bitmap(1024), rb.Bitmap(1024)
    b.set_many([3, 600])
    rb.or_blocks(a, b, 1, 2)
    assert a.to_indices().tolist() == [600]
    rb.copy_blocks(a, b, 0, 1)
    assert a.to_indices().tolist() == [3, 600]


def test_frontier_round_trip():
    rng = np.random.default_rng(12345)
    n = 900
    members = np.unique(rng.integers(0, n, size=50).astype(np.uint32))
    fr = rb.Frontier.from_queue(n, members)
    both = fr.to_bitmap_form()
    assert both.bits.count() == members.size
    back = rb.Frontier.from_bitmap(both.bits)
    assert np.array_equal(back.indices(), members)
    assert back.to_queue_form().count == members.size


def test_scramble_ids_matches_oracle():
    import oracle

    rng = np.random.default_rng(4)
    for scale, seed in ((6, 3), (13, 5), (22, 1), (26, 1)):
        ids = rng.integers(0, 1 << scale, size=1000, dtype=np.uint64)
        assert np.array_equal(rb.scramble_ids(ids, scale, seed), oracle.scramble_ids(ids, scale, seed))
        # a bijection on [0, 2^scale)
        if scale <= 13:
            allv = rb.scramble_ids(np.arange(1 << scale, dtype=np.uint64), scale, seed)
            assert np.unique(allv).size == 1 << scale


def test_sample_sources_convention(golden_kron):
    import oracle

    c = oracle.build_csr(*oracle.kronecker_generate(12))
    g2 = oracle.apply_permutation(c, oracle.rcm(c)[0])
    got = rb.sample_sources(g2.degrees, 16, 1)
    assert got.tolist() == [r["source"] for r in golden_kron["12,1"]["roots"]]


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rcmbfs_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rb_[a-z0-9_]+)\s*\(", src)))


def test_abi_library_exports_header_symbols():
    path = _build.build()
    lib = ctypes.CDLL(path)
    names = _header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)
    L = _lib.load()
    assert L.rb_version() == 1
    # pure host queries work without a GPU
    assert L.rb_csr_workspace_bytes(1000, 100) > 16000
    assert L.rb_rcm_workspace_bytes(1000, 5000) > 0


def test_host_fill_streaming_stores():
    """rb_host_fill_i32 (the -1 tail of BfsResult.predecessor, engine.py:598):
    unaligned starts, lengths around the 16-entry unroll, one and several threads."""
    L = _lib.load()
    rng = np.random.default_rng(5)
    for n, off, threads in [(0, 0, 1), (1, 1, 1), (15, 3, 4), (16, 0, 1), (17, 2, 8), (1000, 1, 2),
                            ((3 << 20) + 5, 3, 4), ((2 << 20), 0, 8)]:
        a = rng.integers(0, 100, size=n + off + 7, dtype=np.int32)
        want = a.copy()
        want[off:off + n] = -1
        rc = L.rb_host_fill_i32(ctypes.c_void_p(a.ctypes.data + 4 * off), n, -1, threads)
        assert rc == 0 and np.array_equal(a, want), (n, off, threads)
    assert L.rb_host_fill_i32(None, 10, -1, 1) != 0  # RB_ERR_ARG
    assert b"rb_host_fill_i32" in L.rb_last_error()


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    el = rb.EdgeList(4, np.array([[0, 1], [1, 2]], np.uint32))
    with pytest.raises(RuntimeError, match="CUDA"):
        rb.build_csr(el)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2012_10026_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_result_pool_never_hands_out_a_live_buffer():
    """Large predecessor arrays come from a pool of mappings (engine.fresh_int32):
    a mapping is reused only after every view of its previous array is gone."""
    import gc

    from paper_2012_10026_b200 import engine

    n = 9 << 20
    a = engine.fresh_int32(n)
    a[:] = 7
    view = a[100:200]
    del a
    gc.collect()
    b = engine.fresh_int32(n)
    assert not np.shares_memory(b, view)
    assert (view == 7).all()
    b[:] = 1
    assert (view == 7).all()
    del view, b
    gc.collect()
    c = engine.fresh_int32(n)  # now a pooled (warm) mapping may come back
    assert c.flags.writeable and c.size == n and c.dtype == np.int32


def test_s29_memory_plan_fits_b200():
    """configs[3] dry run: every stage of the sharded scale-29 pipeline fits one
    B200's HBM at 8 GPUs (sharded.memory_plan), and would not at 2."""
    from paper_2012_10026_b200.sharded import memory_plan, owner_bounds

    plan = memory_plan(29, 8)
    assert plan["fits"], plan
    assert plan["stages_gb"]["rcm_on_root"] == max(plan["stages_gb"].values())
    assert not memory_plan(29, 2)["fits"] or memory_plan(29, 2)["peak_gb"] > 100
    b = owner_bounds(1 << 29, 8)
    assert b[0] == 0 and b[-1] == 1 << 29 and all(x % 8192 == 0 for x in b[:-1]) and len(b) == 9
