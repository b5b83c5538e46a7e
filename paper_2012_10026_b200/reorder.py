"""RCM relabelling, permutation apply and degree-sorted adjacency on device
(reference reorder.py:42-280)."""

from __future__ import annotations

import ctypes
import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import CsrGraph

__all__ = [
    "Permutation",
    "RcmRunStats",
    "rcm",
    "partial_rcm",
    "apply_permutation",
    "degree_sort_adjacency",
    "graph_hash",
]


class Permutation:
    """``perm[new_id] = original_id`` and its inverse (reorder.py:42-68).

    Host numpy arrays are materialized lazily from the device copies."""

    def __init__(self, perm=None, inv=None, *, _dev=None):
        self._perm = None if perm is None else np.ascontiguousarray(perm, dtype=np.uint32)
        self._inv = None if inv is None else np.ascontiguousarray(inv, dtype=np.uint32)
        self._dev = _dev  # (perm, inv) int32 CUDA tensors
        self._size = int(self._perm.size) if self._perm is not None else int(_dev[0].numel())

    @classmethod
    def from_new_to_orig(cls, perm: np.ndarray, check: bool = True) -> "Permutation":
        perm = np.ascontiguousarray(perm, dtype=np.uint32)
        n = perm.size
        if check and n:
            counts = np.bincount(perm, minlength=n)
            if counts.size != n or not np.all(counts == 1):
                raise ValueError("permutation array is not a bijection on [0, n)")
        inv = np.empty(n, dtype=np.uint32)
        inv[perm] = np.arange(n, dtype=np.uint32)
        return cls(perm, inv)

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        ids = np.arange(n, dtype=np.uint32)
        return cls(ids, ids.copy())

    @property
    def perm(self) -> np.ndarray:
        if self._perm is None:
            self._perm = self._dev[0].cpu().numpy().view(np.uint32)
        return self._perm

    @property
    def inv(self) -> np.ndarray:
        if self._inv is None:
            self._inv = self._dev[1].cpu().numpy().view(np.uint32)
        return self._inv

    def device_arrays(self):
        if self._dev is None:
            torch = _lib.require_cuda()
            self._dev = (
                torch.from_numpy(self._perm.view(np.int32)).cuda(),
                torch.from_numpy(self._inv.view(np.int32)).cuda(),
            )
        return self._dev

    @property
    def size(self) -> int:
        return self._size


@dataclass
class RcmRunStats:
    """Component layout of the relabelling traversal (reorder.py:71-103)."""

    n: int
    n_non_isolated: int
    n_assigned: int
    component_ranges: list = field(default_factory=list)

    @property
    def n_components(self) -> int:
        return len(self.component_ranges)

    @property
    def component_sizes(self) -> np.ndarray:
        return np.array([e - s for s, e in self.component_ranges], dtype=np.int64)

    @property
    def largest_component_fraction(self) -> float:
        if self.n_non_isolated == 0 or not self.component_ranges:
            return 0.0
        return float(self.component_sizes.max()) / self.n_non_isolated

    @property
    def complete(self) -> bool:
        return self.n_assigned == self.n_non_isolated


def rcm(g: CsrGraph) -> tuple[Permutation, RcmRunStats]:
    """Full reverse Cuthill-McKee relabelling, bit-exact with reorder.py:231-237.

    Non-isolated vertices occupy new ids [0, |V+|), isolated ones follow in
    ascending original id."""
    torch = _lib.require_cuda()
    L = _lib.lib()
    rs, col, deg = g.device_arrays()
    n = g.n
    ws_bytes = L.rb_rcm_workspace_bytes(n, g.m_directed)
    ws = _lib.workspace(ws_bytes)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    inv = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    ranges = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
    n_plus = ctypes.c_int64(0)
    nc = ctypes.c_int64(0)
    rc = L.rb_rcm(
        _lib.ptr(rs), _lib.ptr(col), _lib.ptr(deg), n, _lib.ptr(ws), ws_bytes, _lib.ptr(perm), _lib.ptr(inv),
        ctypes.byref(n_plus), _lib.ptr(ranges), ctypes.byref(nc), _lib.stream_ptr(),
    )
    _lib.check(rc, "rcm")
    del ws
    rr = ranges[: 2 * nc.value].cpu().numpy().reshape(-1, 2)
    stats = RcmRunStats(
        n=n, n_non_isolated=n_plus.value, n_assigned=n_plus.value,
        component_ranges=[(int(a), int(b)) for a, b in rr],
    )
    return Permutation(_dev=(perm, inv)), stats


def partial_rcm(g: CsrGraph, p: float) -> tuple[Permutation, RcmRunStats]:
    """RCM truncated after ``ceil(p * |V+|)`` labels (reorder.py:240-251);
    ``p = 1`` is exactly :func:`rcm`.

    The truncated walk labels the first k vertices of the full Cuthill-McKee
    order, so on device the partial permutation is the full one's slice
    ``perm[|V+| - k : |V+|]`` (the reversed prefix), then the unlabelled
    non-isolated vertices in ascending original id, then the isolated tail
    (reorder.py:219-220).  Components whose discovery started before k keep
    their ranges, the last one cut at k."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    torch = _lib.require_cuda()
    full, st = rcm(g)
    n, n_plus = g.n, st.n_non_isolated
    k = min(math.ceil(p * n_plus), n_plus)
    if k == n_plus:
        return full, st
    fp, _ = full.device_arrays()
    deg = g.device_arrays()[2]
    placed = torch.zeros(max(n, 1), dtype=torch.bool, device="cuda")
    pre = fp[n_plus - k: n_plus]
    placed[pre.long()] = True
    rest = torch.nonzero((deg > 0) & ~placed[:n]).reshape(-1).to(torch.int32)  # ascending id
    perm = torch.cat([pre, rest, fp[n_plus:]])
    inv = torch.empty_like(perm)
    inv[perm.long()] = torch.arange(n, dtype=torch.int32, device="cuda")
    ranges = []
    for a, b in st.component_ranges:  # full new-id range (a, b) = discovery [n_plus - b, n_plus - a)
        ds, de = n_plus - b, n_plus - a
        if ds < k:
            ranges.append((k - min(de, k), k - ds))
    ranges.sort()
    stats = RcmRunStats(n=n, n_non_isolated=n_plus, n_assigned=k, component_ranges=ranges if k else [])
    return Permutation(_dev=(perm, inv)), stats


def apply_permutation(g: CsrGraph, perm: Permutation) -> CsrGraph:
    """Relabel ``g`` (new vertex i = old perm[i]); rows ascending (reorder.py:254-271)."""
    if perm.size != g.n:
        raise ValueError(f"permutation size {perm.size} != graph size {g.n}")
    torch = _lib.require_cuda()
    L = _lib.lib()
    rs, col, deg = g.device_arrays()
    p, inv = perm.device_arrays()
    n, m = g.n, g.m_directed
    ws_bytes = L.rb_permute_workspace_bytes(n, m)
    ws = _lib.workspace(ws_bytes)
    rs2 = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col2 = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")[:m]
    deg2 = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    rc = L.rb_apply_permutation(
        _lib.ptr(rs), _lib.ptr(col), _lib.ptr(deg), n, m, _lib.ptr(p), _lib.ptr(inv), _lib.ptr(ws), ws_bytes,
        _lib.ptr(rs2), _lib.ptr(col2), _lib.ptr(deg2), _lib.stream_ptr(),
    )
    _lib.check(rc, "apply_permutation")
    return CsrGraph(n, _dev=(rs2, col2, deg2))


def degree_sort_adjacency(g: CsrGraph, order: str = "descending") -> CsrGraph:
    """Rows re-sorted by neighbour degree, ties by ascending id (reorder.py:181-195)."""
    if order not in ("ascending", "descending"):
        raise ValueError(f"order must be 'ascending' or 'descending', got {order!r}")
    torch = _lib.require_cuda()
    L = _lib.lib()
    rs, col, deg = g.device_arrays()
    n, m = g.n, g.m_directed
    ws_bytes = L.rb_permute_workspace_bytes(n, m)
    ws = _lib.workspace(ws_bytes)
    col2 = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")[:m]
    if m:
        rc = L.rb_degree_sort_adjacency(
            _lib.ptr(rs), _lib.ptr(col), _lib.ptr(deg), n, m, int(order == "descending"), _lib.ptr(ws), ws_bytes,
            _lib.ptr(col2), _lib.stream_ptr(),
        )
        _lib.check(rc, "degree_sort_adjacency")
    return CsrGraph(n, _dev=(rs, col2, deg))


def graph_hash(g: CsrGraph) -> str:
    """sha256 over the canonical CSR arrays (reorder.py:274-280)."""
    h = hashlib.sha256()
    h.update(np.int64(g.n).tobytes())
    h.update(np.ascontiguousarray(g.row_starts).tobytes())
    h.update(np.ascontiguousarray(g.dst).tobytes())
    return h.hexdigest()
