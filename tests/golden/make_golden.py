"""Generate golden fixtures by running the REFERENCE package (rcmbfs).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes small files next to this script; they are committed and read by the
tests (CPU: oracle pinning; GPU: device parity).  Nothing here is imported by
the product package.

Contents
* generator.json  -- sha256 of kronecker_generate edges + CSR counts per params
* small.npz       -- random multigraphs: edges, RCM perm, component ranges,
                     sequential parents/levels for a few sources, step results
* kron.json       -- per (scale, seed): RCM perm sha256, component count,
                     |V+|, 64 (or fewer) _sample_sources roots with per-root
                     level-array sha256, hybrid LevelRecord tuples
                     (direction, n_f, m_f, m_u), traversed edges, raw pairs
* kron12_perm.npy -- full RCM permutation of Kronecker scale 12 seed 1
* validate.npz    -- the reference Validator on random graphs with randomly
                     corrupted trees (cycles, phantom edges, dropped and
                     foreign vertices): check vector, details, derived levels
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import rcmbfs
from rcmbfs import (
    BfsParams,
    Bitmap,
    EdgeList,
    Frontier,
    KroneckerParams,
    Validator,
    apply_permutation,
    bfs_run,
    bfs_sequential,
    bottom_up_step,
    build_csr,
    kronecker_generate,
    rcm,
    top_down_step,
)
from rcmbfs.bench import _sample_sources

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_fixtures():
    out = {}
    for scale, ef, seed in [(6, 4, 3), (10, 16, 42), (13, 16, 5), (14, 16, 9), (16, 16, 1), (16, 16, 7)]:
        el = kronecker_generate(KroneckerParams(scale=scale, edgefactor=ef, seed=seed))
        g = build_csr(el)
        out[f"{scale},{ef},{seed}"] = {
            "edges_sha256": sha(el.edges),
            "m_directed": g.m_directed,
            "isolated": g.isolated_count,
            "row_starts_sha256": sha(g.row_starts),
            "dst_sha256": sha(g.dst),
        }
        print("gen", scale, ef, seed, g.m_directed, g.isolated_count, flush=True)
    with open(os.path.join(HERE, "generator.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def small_fixtures():
    rng = np.random.default_rng(2024)
    arrays = {}
    meta = []
    for gi in range(24):
        n = int(rng.integers(2, 1500))
        density = float(rng.choice([0.3, 1.0, 2.5, 4.0]))
        m = max(1, int(n * density))
        e = rng.integers(0, n, size=(m, 2), dtype=np.uint32)
        el = EdgeList(n_declared=n, edges=e)
        g = build_csr(el)
        perm, st = rcm(g)
        g2 = apply_permutation(g, perm)
        arrays[f"g{gi}_edges"] = e
        arrays[f"g{gi}_perm"] = perm.perm
        arrays[f"g{gi}_ranges"] = np.array(st.component_ranges, dtype=np.int64).reshape(-1, 2)
        arrays[f"g{gi}_rcm_dst"] = g2.dst
        srcs = rng.choice(n, size=min(4, n), replace=False)
        val = Validator(g2)
        lev = []
        for s in srcs:
            r = bfs_sequential(g2, int(s))
            rep = val.validate(int(s), r.predecessor)
            assert rep.passed
            lev.append(rep.derived_levels.astype(np.int32))
            arrays[f"g{gi}_seqpar_{int(s)}"] = r.predecessor
        arrays[f"g{gi}_srcs"] = srcs.astype(np.int64)
        arrays[f"g{gi}_levels"] = np.stack(lev)
        # one TD and one BU reference step from a random state (criterion 2 style)
        vis_mask = rng.random(n) < 0.3
        vis_mask[int(srcs[0])] = True
        vis_idx = np.flatnonzero(vis_mask)
        f_idx = vis_idx[rng.random(vis_idx.size) < 0.5]
        if f_idx.size == 0:
            f_idx = vis_idx[:1]
        for kind, fn in (("td", top_down_step), ("bu", bottom_up_step)):
            visited = Bitmap.from_indices(n, vis_idx)
            parent = np.full(n, -1, np.int32)
            parent[vis_idx] = vis_idx
            fr = Frontier.from_queue(n, f_idx.astype(np.uint32))
            nxt, stats = fn(g2, fr, visited, parent)
            arrays[f"g{gi}_{kind}_next"] = np.sort(nxt.indices()).astype(np.uint32)
            arrays[f"g{gi}_{kind}_visited"] = visited.words.copy()
            arrays[f"g{gi}_{kind}_stats"] = np.array([stats.n_next, stats.deg_next, stats.scanned_edges], np.int64)
        arrays[f"g{gi}_state_vis"] = vis_idx.astype(np.int64)
        arrays[f"g{gi}_state_frontier"] = f_idx.astype(np.int64)
        meta.append(n)
    arrays["n_list"] = np.array(meta, np.int64)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    print("small fixtures", len(meta), flush=True)


def kron_fixtures(plan):
    out = {}
    for scale, seed, n_roots in plan:
        el = kronecker_generate(KroneckerParams(scale=scale, edgefactor=16, seed=seed))
        g = build_csr(el)
        perm, st = rcm(g)
        g2 = apply_permutation(g, perm)
        if scale == 12 and seed == 1:
            np.save(os.path.join(HERE, "kron12_perm.npy"), perm.perm)
        relabeled = EdgeList(n_declared=g2.n, edges=perm.inv[el.edges.reshape(-1)].reshape(-1, 2))
        val = Validator(g2, edge_list=relabeled)
        labels = val.component_labels()
        raw_per_label = np.bincount(labels[relabeled.edges[:, 0]], minlength=g2.n)
        srcs = _sample_sources(g2, n_roots, 1)
        roots = []
        for s in srcs:
            s = int(s)
            res = bfs_run(g2, s, BfsParams(mode="hybrid", alpha=64, beta=8))
            rep = val.validate(s, res.predecessor)
            assert rep.passed
            roots.append(
                {
                    "source": s,
                    "levels_sha256": sha(rep.derived_levels.astype(np.int32)),
                    "records": [
                        ["T" if r.direction == rcmbfs.TOP_DOWN else "B", r.n_f, r.m_f, r.m_u]
                        for r in res.levels
                    ],
                    "traversed": int(res.traversed_edges),
                    "raw_pairs": int(raw_per_label[labels[s]]),
                    "n_reached": int(res.n_reached),
                }
            )
        out[f"{scale},{seed}"] = {
            "n": g.n,
            "m_directed": g.m_directed,
            "n_plus": int(g.n - g.isolated_count),
            "perm_sha256": sha(perm.perm),
            "rcm_dst_sha256": sha(g2.dst),
            "rcm_row_starts_sha256": sha(g2.row_starts),
            "n_components": st.n_components,
            "component_ranges_sha256": sha(np.array(st.component_ranges, np.int64)),
            "largest_component_fraction": st.largest_component_fraction,
            "roots": roots,
        }
        print("kron", scale, seed, g.m_directed, st.n_components, flush=True)
    return out


def validate_fixtures():
    """Reference Validator (validate.py:123-225) on corrupted predecessor arrays."""
    rng = np.random.default_rng(2024)
    arrays = {}
    details = []
    i = 0
    for gi in range(12):
        n = int(rng.integers(8, 700))
        e = rng.integers(0, n, size=(int(n * rng.choice([0.6, 1.2, 3.0])), 2), dtype=np.uint32)
        g = build_csr(EdgeList(n_declared=n, edges=e))
        val = Validator(g)
        src = int(rng.integers(0, n))
        base = bfs_sequential(g, src).predecessor.astype(np.int32)
        arrays[f"g{gi}_n"] = np.array([n])
        arrays[f"g{gi}_edges"] = e
        for t in range(6):
            bad = base.copy()
            if t == 1:  # 2-cycle between reached neighbours
                reach = np.flatnonzero(base >= 0)
                for a in reach:
                    nb = [int(w) for w in g.neighbors(int(a)) if int(w) != src and base[w] >= 0]
                    if int(a) != src and nb:
                        bad[a], bad[nb[0]] = nb[0], a
                        break
            elif t >= 2:
                k = int(rng.integers(1, 4))
                idx = rng.integers(0, n, size=k)
                bad[idx] = rng.integers(-1, n, size=k)
            rep = val.validate(src, bad)
            arrays[f"c{i}_graph"] = np.array([gi, src])
            arrays[f"c{i}_parent"] = bad
            arrays[f"c{i}_checks"] = np.array([c.passed for c in rep.checks])
            arrays[f"c{i}_levels"] = rep.derived_levels.astype(np.int64)
            details.append([c.detail for c in rep.checks])
            i += 1
    arrays["n_cases"] = np.array([i])
    np.savez_compressed(os.path.join(HERE, "validate.npz"), **arrays)
    with open(os.path.join(HERE, "validate_details.json"), "w") as f:
        json.dump(details, f, indent=0)
    print("validate", i, flush=True)


def mode_fixtures():
    """Full LevelRecords of the partitioned modes (hybrid_balanced: bu_steal;
    hybrid_reduced: Alg. 6 two-pass bu_reduced on the descending adjacency)
    incl. scanned / pass1_hits / live_vertices / claimed, for several thread
    counts and partition factors (engine.py:478-604, partition.py)."""
    from rcmbfs import degree_sort_adjacency

    out = {}
    for scale, seed in ((12, 1), (14, 3), (16, 1)):
        el = kronecker_generate(KroneckerParams(scale=scale, edgefactor=16, seed=seed))
        g = build_csr(el)
        perm, _ = rcm(g)
        g2 = apply_permutation(g, perm)
        gd = degree_sort_adjacency(g2, "descending")
        srcs = [int(s) for s in _sample_sources(g2, 6, 3)]
        cases = []
        for mode in ("hybrid_reduced", "hybrid_balanced"):
            for threads, lam in ((1, 20), (3, 10), (4, 1)):
                params = BfsParams(mode=mode, threads=threads, partition_factor=lam)
                with rcmbfs.BfsEngine(g2, params, g_desc=gd) as eng:
                    for s in srcs:
                        res = eng.run(s)
                        cases.append({
                            "mode": mode, "threads": threads, "partition_factor": lam, "source": s,
                            "records": [["T" if r.direction == rcmbfs.TOP_DOWN else "B", r.n_f, r.m_f, r.m_u,
                                         r.scanned_edges, r.pass1_hits, r.live_vertices, r.claimed]
                                        for r in res.levels],
                        })
        out[f"{scale},{seed}"] = cases
        print("modes", scale, seed, len(cases), flush=True)
    with open(os.path.join(HERE, "modes.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)


def partial_fixtures():
    """partial_rcm (reorder.py:240-251) perms and stats, get_partitions and
    shrink_partition (partition.py:67-178) on random bitmaps."""
    from rcmbfs import get_partitions, partial_rcm, shrink_partition

    out = {"partial": [], "partitions": [], "shrink": []}
    for scale, seed in ((12, 1), (14, 3)):
        g = build_csr(kronecker_generate(KroneckerParams(scale=scale, edgefactor=16, seed=seed)))
        for p in (0.05, 0.3, 0.5, 0.999, 1.0):
            perm, st = partial_rcm(g, p)
            out["partial"].append({"scale": scale, "seed": seed, "p": p, "perm_sha256": sha(perm.perm),
                                   "n_assigned": st.n_assigned, "ranges": [list(r) for r in st.component_ranges]})
    rng = np.random.default_rng(5)
    import warnings
    for n, lam, t in ((1, 1, 1), (511, 2, 2), (512, 1, 1), (10000, 10, 4), (1 << 16, 20, 1), (1 << 16, 10, 16),
                      (123457, 7, 3), (5000, 20, 8)):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ps = get_partitions(n, lam, t)
        out["partitions"].append({"n": n, "factor": lam, "threads": t, "starts": ps.starts.tolist(),
                                  "ends": ps.ends.tolist()})
    for case in range(40):
        n = int(rng.integers(1, 20000))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ps = get_partitions(n, int(rng.integers(1, 8)), int(rng.integers(1, 4)))
        vis = Bitmap(n)
        full_blocks = rng.random(vis.n_blocks) < rng.choice([0.3, 0.8, 1.0])
        idx = np.concatenate([np.arange(b * 512, min(n, (b + 1) * 512)) for b in np.flatnonzero(full_blocks)]
                             + [rng.integers(0, n, size=n // 7)]).astype(np.int64)
        if idx.size:
            vis.set_many(idx)
        res = []
        for i in range(ps.n_partitions):
            res.append(list(shrink_partition(ps, i, vis)))
        out["shrink"].append({"n": n, "starts": ps.starts.tolist(), "ends": ps.ends.tolist(),
                              "set": np.unique(idx).tolist() if idx.size < 3000 else None,
                              "set_sha256": sha(vis.words), "words": vis.words.view(np.uint64).tolist()
                              if vis.words.size <= 400 else None, "result": res})
    with open(os.path.join(HERE, "partial.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("partial", len(out["partial"]), len(out["partitions"]), len(out["shrink"]), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["gen", "small", "kron", "validate"]
    if "validate" in which:
        validate_fixtures()
    if "gen" in which:
        gen_fixtures()
    if "small" in which:
        small_fixtures()
    if "modes" in which:
        mode_fixtures()
    if "partial" in which:
        partial_fixtures()
    if "s22" in which:  # BASELINE configs[1]: appended to kron.json (reference build ~4 min)
        path = os.path.join(HERE, "kron.json")
        with open(path) as f:
            data = json.load(f)
        data.update(kron_fixtures([(22, 1, 8)]))
        with open(path, "w") as f:
            json.dump(data, f, indent=0, sort_keys=True)
    if "kron" in which:
        plan = [(12, 1, 16), (14, 3, 16), (16, 1, 64), (18, 1, 16)]
        if "big" in which:
            plan.append((20, 1, 8))
        data = kron_fixtures(plan)
        with open(os.path.join(HERE, "kron.json"), "w") as f:
            json.dump(data, f, indent=0, sort_keys=True)
