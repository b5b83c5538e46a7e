"""EdgeList / CsrGraph and the device CSR build (reference graph.py:39-142).

``CsrGraph`` keeps the reference's field names (``n``, ``row_starts`` int64,
``dst`` uint32, ``degrees`` int32) but is *device-resident*: arrays produced
by the CUDA pipeline stay in HBM (``row_starts`` int64, ``col`` int32,
``degrees`` int32) and host numpy copies are materialized lazily on first
access.  A graph built from numpy arrays uploads on first device use.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["EdgeList", "CsrGraph", "build_csr", "neighbors", "bandwidth"]


class EdgeList:
    """Raw pairs plus declared vertex count (graph.py:39-52).

    ``edges`` is an (m, 2) uint32 numpy array or a CUDA tensor of the same
    shape (int32/uint32 bit pattern)."""

    def __init__(self, n_declared: int, edges):
        self.n_declared = int(n_declared)
        self.edges = edges

    @property
    def m_raw(self) -> int:
        return int(self.edges.shape[0])

    def __repr__(self) -> str:
        return f"EdgeList(n_declared={self.n_declared}, m_raw={self.m_raw})"


class CsrGraph:
    """Undirected simple graph in CSR form (graph.py:55-82), HBM-resident."""

    def __init__(self, n: int, row_starts=None, dst=None, degrees=None, *, _dev=None):
        self.n = int(n)
        self._rs = None if row_starts is None else np.ascontiguousarray(row_starts, dtype=np.int64)
        self._dst = None if dst is None else np.ascontiguousarray(dst, dtype=np.uint32)
        self._deg = None if degrees is None else np.ascontiguousarray(degrees, dtype=np.int32)
        self._dev = _dev  # (row_starts int64, col int32, degrees int32) CUDA tensors
        self._m = None
        if self._dst is not None:
            self._m = int(self._dst.size)
        elif _dev is not None:
            self._m = int(_dev[1].numel())
        self._cache = {}

    # -- device side ----------------------------------------------------
    def device_arrays(self):
        """(row_starts int64, col int32, degrees int32) CUDA tensors."""
        if self._dev is None:
            torch = _lib.require_cuda()
            rs = torch.from_numpy(self._rs).cuda()
            col = torch.from_numpy(self._dst.view(np.int32)).cuda()
            deg = torch.from_numpy(self._deg).cuda()
            self._dev = (rs, col, deg)
        return self._dev

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    # -- host side (reference fields) -------------------------------------
    def _host(self):
        if self._rs is None:
            rs, col, deg = self._dev
            self._rs = rs.cpu().numpy()
            self._dst = col.cpu().numpy().view(np.uint32)
            self._deg = deg.cpu().numpy()
        return self._rs, self._dst, self._deg

    @property
    def row_starts(self) -> np.ndarray:
        return self._host()[0]

    @property
    def dst(self) -> np.ndarray:
        return self._host()[1]

    @property
    def degrees(self) -> np.ndarray:
        return self._host()[2]

    @property
    def m_directed(self) -> int:
        return int(self._m)

    @property
    def m_undirected(self) -> int:
        return self.m_directed // 2

    @property
    def isolated_count(self) -> int:
        if "iso" not in self._cache:
            if self._deg is None and self._dev is not None:
                self._cache["iso"] = int((self._dev[2] == 0).sum().item())
            else:
                self._cache["iso"] = int(np.count_nonzero(self.degrees == 0))
        return self._cache["iso"]

    def neighbors(self, v: int) -> np.ndarray:
        rs = self.row_starts
        return self.dst[rs[v] : rs[v + 1]]

    def __repr__(self) -> str:
        where = "cuda" if self._dev is not None else "host"
        return f"CsrGraph(n={self.n}, m_directed={self.m_directed}, {where})"


def _edges_device(el: EdgeList):
    torch = _lib.require_cuda()
    e = el.edges
    if isinstance(e, torch.Tensor):
        if e.ndim != 2 or e.shape[1] != 2:
            raise ValueError(f"edge array must have shape (m, 2), got {tuple(e.shape)}")
        return e.contiguous().cuda(), None
    a = np.asarray(e)
    if a.size == 0:
        a = a.reshape(0, 2)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError(f"edge array must have shape (m, 2), got {a.shape}")
    if a.dtype != np.uint32:
        a64 = a.astype(np.int64)
        if a64.size and (a64.min() < 0 or a64.max() >= 1 << 32):
            # negative / >32-bit ids cannot be stored; report like graph.py:103-108
            bad = np.flatnonzero((a64[:, 0] < 0) | (a64[:, 0] >= el.n_declared) | (a64[:, 1] < 0) | (a64[:, 1] >= el.n_declared))
            i = int(bad[0])
            raise ValueError(f"edge {i} = ({int(a64[i, 0])}, {int(a64[i, 1])}) out of range for n={el.n_declared}")
        a = a64.astype(np.uint32)
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a.view(np.int32)).cuda(non_blocking=False)
    return t, a


def build_csr(el: EdgeList) -> CsrGraph:
    """Canonicalize an edge list on the device (graph.py:85-120).

    Symmetrizes, drops self-loops, deduplicates and sorts rows ascending;
    raises ``ValueError`` naming the first out-of-range edge."""
    n = int(el.n_declared)
    if n < 0:
        raise ValueError(f"vertex count must be non-negative, got {n}")
    torch = _lib.require_cuda()
    L = _lib.lib()
    ed, host = _edges_device(el)
    m = int(ed.shape[0])
    ws_bytes = L.rb_csr_workspace_bytes(m, n)
    ws = _lib.workspace(ws_bytes)
    md = ctypes.c_int64(0)
    bad = ctypes.c_int64(-1)
    s = _lib.stream_ptr()
    rc = L.rb_csr_build(_lib.ptr(ed), m, n, _lib.ptr(ws), ws_bytes, ctypes.byref(md), ctypes.byref(bad), s)
    if rc == _lib.RB_ERR_ARG and bad.value >= 0:
        i = bad.value
        row = host[i] if host is not None else ed[i].cpu().numpy().view(np.uint32)
        u, v = int(row[0]), int(row[1])
        raise ValueError(f"edge {i} = ({u}, {v}) out of range for n={n}")
    _lib.check(rc, "build_csr")
    rs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(max(md.value, 1), dtype=torch.int32, device="cuda")[: md.value]
    deg = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    _lib.check(L.rb_csr_emit(_lib.ptr(ws), md.value, n, _lib.ptr(rs), _lib.ptr(col), _lib.ptr(deg), s), "csr_emit")
    del ws
    return CsrGraph(n, _dev=(rs, col, deg))


def neighbors(g: CsrGraph, v: int) -> np.ndarray:
    return g.neighbors(v)


def bandwidth(g: CsrGraph) -> int:
    """max |u - v| over stored edges (graph.py:128-142), computed on device."""
    if g.m_directed == 0:
        return 0
    torch = _lib.require_cuda()
    rs, col, deg = g.device_arrays()
    src = torch.repeat_interleave(torch.arange(g.n, device="cuda", dtype=torch.int64), deg.to(torch.int64))
    return int((src - col.to(torch.int64)).abs().max().item())
