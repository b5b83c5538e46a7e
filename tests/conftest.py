"""Shared fixtures.  The oracle (CPU restatement of the reference) is the
checker; the product package is what is tested.  GPU tests are marked
``@pytest.mark.gpu`` and call through the C ABI."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger sizes")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="session")
def golden_gen():
    with open(os.path.join(GOLDEN, "generator.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_kron():
    with open(os.path.join(GOLDEN, "kron.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(os.path.join(GOLDEN, "small.npz")))


class OracleCache:
    """Session cache of oracle-built Kronecker graphs: (n, edges, csr, perm, csr_rcm)."""

    def __init__(self):
        self._s = {}

    def kron(self, scale, seed=1, ef=16):
        key = (scale, seed, ef)
        if key not in self._s:
            import oracle

            n, e = oracle.kronecker_generate(scale, ef, seed=seed)
            g = oracle.build_csr(n, e)
            perm, k, ranges = oracle.rcm(g)
            g2 = oracle.apply_permutation(g, perm)
            self._s[key] = dict(n=n, edges=e, g=g, perm=perm, n_plus=k, ranges=ranges, g2=g2)
        return self._s[key]


@pytest.fixture(scope="session")
def ocache():
    return OracleCache()


def small_graph(golden_small, i):
    import oracle

    n = int(golden_small["n_list"][i])
    e = golden_small[f"g{i}_edges"]
    return n, e


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


@pytest.fixture(scope="session")
def golden_validate():
    arr = dict(np.load(os.path.join(GOLDEN, "validate.npz")))
    with open(os.path.join(GOLDEN, "validate_details.json")) as f:
        details = json.load(f)
    return arr, details


def validate_cases(golden):
    """Yield (n, edges, source, parent, checks, levels, details) per reference case."""
    arr, details = golden
    for i in range(int(arr["n_cases"][0])):
        gi, src = (int(x) for x in arr[f"c{i}_graph"])
        yield (int(arr[f"g{gi}_n"][0]), arr[f"g{gi}_edges"], src, arr[f"c{i}_parent"], arr[f"c{i}_checks"].tolist(),
               arr[f"c{i}_levels"], details[i])


@pytest.fixture(scope="session")
def golden_modes():
    with open(os.path.join(GOLDEN, "modes.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_partial():
    with open(os.path.join(GOLDEN, "partial.json")) as f:
        return json.load(f)


def mode_records(recs_or_rows, from_oracle: bool):
    """[dir, n_f, m_f, m_u, scanned, pass1_hits, live_vertices, claimed] rows
    (None for the reference's absent fields) from oracle rows or LevelRecords."""
    out = []
    for r in recs_or_rows:
        if from_oracle:
            d, nf, mf, mu, sc, p1, lv, cl = (int(x) for x in r[1:9])
            out.append(["T" if d == 0 else "B", nf, mf, mu, sc, None if p1 < 0 else p1, None if lv < 0 else lv,
                        None if cl < 0 else cl])
        else:
            out.append(["T" if r.direction == "top_down" else "B", r.n_f, r.m_f, r.m_u, r.scanned_edges,
                        r.pass1_hits, r.live_vertices, r.claimed])
    return out
