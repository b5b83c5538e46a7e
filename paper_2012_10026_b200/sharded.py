"""Sharded preprocessing for graphs that do not fit one GPU's working set
(BASELINE configs[3]: Kronecker scale 29, ~17 B directed CSR entries, 8 B200).

The single-GPU pipeline (generate -> build_csr -> rcm -> apply_permutation,
graph.py:85-120 / reorder.py:198-271) needs the raw edges, 2 x m sort keys and
the whole CSR in one HBM.  Here every step that touches all edges is split by
vertex block over the ranks (one process per GPU, torch.distributed):

1. generate: rank r draws its share of the 65,536-edge chunks on device
   (rb_kronecker_generate_range -- the same Philox streams, so the union is
   byte-identical with kronecker_generate);
2. build: both orientations of its pairs become keys u << 32 | v, sorted and
   deduplicated locally (rb_csr_build), routed to the owner of u (equal
   8192-aligned blocks of the scrambled original ids) with one all-to-all,
   merged and deduplicated again (rb_keys_sort_unique) and turned into the
   block's CSR rows (rb_keys_to_csr) -- exactly graph.py's np.unique, by block;
3. RCM: the rows are gathered on one rank, whose HBM holds the whole CSR plus
   the RCM workspace (scale 29: ~75 GB + ~45 GB of 180 GB, see
   ``memory_plan``), and rcm() runs there unchanged (bit-exact walk order);
   the inverse permutation is broadcast;
4. relabel: every rank maps its rows to keys inv[v] << 32 | inv[w]
   (rb_relabel_keys), routes them to the owners of the new ids (edge-balanced
   blocks of the RCM id range, distributed.partition_bounds) and builds its
   block of the relabelled CSR -- apply_permutation by block, rows ascending.

The result feeds the 1D-partitioned traversal (distributed.DevicePartition /
GpuLocalLevel.from_rows).  Collectives go through NCCL, or through host
memory when the group is gloo (the CPU / one-GPU tests).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .generator import CHUNK_EDGES, KroneckerParams

__all__ = ["LocalRows", "owner_bounds", "sharded_kronecker_csr", "gather_rows_to_root", "relabel_sharded",
           "build_sharded_rcm_graph", "memory_plan"]

BLOCK_ALIGN = 8192


@dataclass
class LocalRows:
    """CSR rows of the vertex block [lo, hi) of an n-vertex graph, columns in
    global ids; rs starts at 0 (int64, hi - lo + 1), col int32, deg int32 --
    CUDA tensors."""

    n: int
    lo: int
    hi: int
    rs: object
    col: object
    deg: object

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    @property
    def m_local(self) -> int:
        return int(self.col.numel())


def owner_bounds(n: int, world: int, align: int = BLOCK_ALIGN) -> list[int]:
    """Equal, align-multiple vertex blocks of the original id range (the
    generator scrambles ids, so equal blocks carry equal expected degree)."""
    per = -(-n // world)
    per = -(-per // align) * align
    return [min(r * per, n) for r in range(world)] + [n]


def _view(ptr: int, n: int, typestr: str):
    import torch

    class _H:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_H(), device="cuda")


def _host_staged(group) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def _all_to_all(send, splits_send, group):
    """Variable-size all-to-all of a 1-D CUDA tensor (counts exchanged first)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    stage = _host_staged(group)
    cnt = torch.tensor(splits_send, dtype=torch.int64)
    cnt_recv = torch.empty(world, dtype=torch.int64)
    if stage:
        dist.all_to_all_single(cnt_recv, cnt, group=group)
    else:
        cr = cnt_recv.cuda()
        dist.all_to_all_single(cr, cnt.cuda(), group=group)
        cnt_recv = cr.cpu()
    splits_recv = [int(x) for x in cnt_recv]
    if stage:
        recv = torch.empty(sum(splits_recv), dtype=send.dtype)
        dist.all_to_all_single(recv, send.cpu(), splits_recv, list(splits_send), group=group)
        return recv.cuda()
    recv = torch.empty(sum(splits_recv), dtype=send.dtype, device="cuda")
    dist.all_to_all_single(recv, send, splits_recv, list(splits_send), group=group)
    return recv


def _sort_unique(keys, end_bit: int):
    import torch

    L = _lib.lib()
    m = int(keys.numel())
    wsb = L.rb_keys_workspace_bytes(m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    mo = ctypes.c_int64(0)
    _lib.check(L.rb_keys_sort_unique(_lib.ptr(keys), m, end_bit, _lib.ptr(ws), wsb, ctypes.byref(mo),
                                     _lib.stream_ptr()), "rb_keys_sort_unique")
    return keys[: mo.value]


def _rows_from_keys(keys, n: int, lo: int, hi: int) -> LocalRows:
    import torch

    m = int(keys.numel())
    rs = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")[:m]
    deg = torch.empty(max(hi - lo, 1), dtype=torch.int32, device="cuda")[: hi - lo]
    _lib.check(_lib.lib().rb_keys_to_csr(_lib.ptr(keys), m, lo, hi - lo, _lib.ptr(rs), _lib.ptr(col), _lib.ptr(deg),
                                          _lib.stream_ptr()), "rb_keys_to_csr")
    return LocalRows(n, lo, hi, rs, col, deg)


def _split_by_owner(keys, bounds: list[int]) -> list[int]:
    """Sizes of the owner segments of sorted keys (owner of key = block of key >> 32)."""
    import torch

    edges = torch.tensor([b << 32 for b in bounds[1:-1]], dtype=torch.int64, device="cuda")
    cut = torch.searchsorted(keys, edges).cpu().tolist() if len(bounds) > 2 else []
    pos = [0] + cut + [int(keys.numel())]
    return [pos[i + 1] - pos[i] for i in range(len(pos) - 1)]


def _bits(x: int) -> int:
    return max(1, int(x).bit_length())


def sharded_kronecker_csr(params: KroneckerParams, rank: int, world: int, group=None) -> LocalRows:
    """Steps 1-2: this rank's block of build_csr(kronecker_generate(params))."""
    import torch

    params.validate()
    L = _lib.lib()
    n, m = params.n, params.m
    chunks = -(-m // CHUNK_EDGES)
    c0, c1 = chunks * rank // world, chunks * (rank + 1) // world
    e_lo, e_hi = min(c0 * CHUNK_EDGES, m), min(c1 * CHUNK_EDGES, m)
    edges = torch.empty((max(e_hi - e_lo, 1), 2), dtype=torch.int32, device="cuda")[: e_hi - e_lo]
    a, b, c, _ = params.initiator
    _lib.check(L.rb_kronecker_generate_range(params.scale, params.edgefactor, params.seed, float(a), float(b),
                                             float(c), e_lo, e_hi, _lib.ptr(edges), _lib.stream_ptr()),
               "rb_kronecker_generate_range")
    m_loc = e_hi - e_lo
    wsb = L.rb_csr_workspace_bytes(m_loc, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    md, bad = ctypes.c_int64(0), ctypes.c_int64(-1)
    _lib.check(L.rb_csr_build(_lib.ptr(edges), m_loc, n, _lib.ptr(ws), wsb, ctypes.byref(md), ctypes.byref(bad),
                              _lib.stream_ptr()), "rb_csr_build")
    del edges
    kp = ctypes.c_void_p(0)
    mk = ctypes.c_int64(0)
    _lib.check(L.rb_csr_keys(_lib.ptr(ws), ctypes.byref(kp), ctypes.byref(mk)), "rb_csr_keys")
    keys = _view(kp.value, mk.value, "<i8")  # sorted unique (u << 32 | v), u < 2^31: signed order = unsigned
    bounds = owner_bounds(n, world)
    recv = _all_to_all(keys.contiguous(), _split_by_owner(keys, bounds), group)
    del ws, keys
    recv = _sort_unique(recv, 32 + _bits(n - 1))
    return _rows_from_keys(recv, n, bounds[rank], bounds[rank + 1])


def gather_rows_to_root(rows: LocalRows, world: int, root: int = 0, group=None):
    """Step 3a: the whole CSR (CsrGraph) on ``root`` (None elsewhere); blocks
    arrive in rank order, so row starts are one running sum."""
    import torch
    import torch.distributed as dist

    from .graph import CsrGraph

    rank = dist.get_rank(group)
    stage = _host_staged(group)
    sizes = [None] * world
    dist.all_gather_object(sizes, (rows.lo, rows.hi, rows.m_local), group=group)
    if rank != root:
        for t in (rows.deg, rows.col):
            dist.send(t.cpu() if stage else t.contiguous(), dst=root, group=group)
        return None
    n = rows.n
    deg = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    m_tot = sum(s[2] for s in sizes)
    col = torch.empty(max(m_tot, 1), dtype=torch.int32, device="cuda")[:m_tot]
    off = 0
    for q, (lo, hi, mq) in enumerate(sizes):
        if q == root:
            deg[lo:hi] = rows.deg
            col[off: off + mq] = rows.col
        else:
            for dst_t in (deg[lo:hi], col[off: off + mq]):
                buf = torch.empty(dst_t.numel(), dtype=torch.int32, device="cpu" if stage else "cuda")
                dist.recv(buf, src=q, group=group)
                dst_t.copy_(buf)
        off += mq
    rs = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(deg.to(torch.int64), 0, out=rs[1:])
    return CsrGraph(n, _dev=(rs, col, deg))


def relabel_sharded(rows: LocalRows, inv, new_bounds: list[int], rank: int, group=None) -> LocalRows:
    """Step 4: this rank's block [new_bounds[rank], new_bounds[rank + 1]) of
    apply_permutation(g, perm), from every rank's old-id rows."""
    import torch

    m = rows.m_local
    keys = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")[:m]
    _lib.check(_lib.lib().rb_relabel_keys(_lib.ptr(rows.rs), _lib.ptr(rows.col), rows.n_local, rows.lo,
                                          _lib.ptr(inv), _lib.ptr(keys), _lib.stream_ptr()), "rb_relabel_keys")
    keys = _sort_unique(keys, 32 + _bits(rows.n - 1))
    recv = _all_to_all(keys, _split_by_owner(keys, new_bounds), group)
    recv = _sort_unique(recv, 32 + _bits(rows.n - 1))
    return _rows_from_keys(recv, rows.n, new_bounds[rank], new_bounds[rank + 1])


def build_sharded_rcm_graph(params: KroneckerParams, rank: int, world: int, group=None, root: int = 0):
    """Steps 1-4.  Returns (this rank's block of the RCM graph as LocalRows,
    the edge-balanced new-id bounds, RcmRunStats, m_directed, perm on root
    (numpy) or None)."""
    import torch
    import torch.distributed as dist

    from .distributed import ALIGN, partition_bounds
    from .reorder import rcm

    rows = sharded_kronecker_csr(params, rank, world, group)
    g = gather_rows_to_root(rows, world, root, group)
    n = rows.n
    obj = [None]
    perm_np = None
    if rank == root:
        perm, stats = rcm(g)
        inv = perm.device_arrays()[1]
        deg_new = g.device_arrays()[2][perm.device_arrays()[0].long()]
        rs_new = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        torch.cumsum(deg_new.to(torch.int64), 0, out=rs_new[1:])
        bounds = partition_bounds(rs_new.cpu().numpy(), stats.n_non_isolated, world, ALIGN)
        obj = [(bounds, stats, g.m_directed)]
        perm_np = perm.perm
        del g, deg_new, rs_new
    else:
        inv = torch.empty(n, dtype=torch.int32, device="cuda")
    dist.broadcast_object_list(obj, src=root, group=group)
    bounds, stats, m_directed = obj[0]
    if _host_staged(group):
        h = inv.cpu()
        dist.broadcast(h, src=root, group=group)
        inv = h.cuda()
    else:
        dist.broadcast(inv, src=root, group=group)
    new_rows = relabel_sharded(rows, inv, bounds, rank, group)
    return new_rows, bounds, stats, m_directed, perm_np


def memory_plan(scale: int = 29, world: int = 8, edgefactor: int = 16, hbm_gb: float = 178.0,
                directed_per_raw: float = 1.99, nonisolated_frac: float = 0.42) -> dict:
    """Per-GPU peak bytes of every stage at ``scale`` over ``world`` GPUs (the
    s29 dry run).  Ratios: m_directed / m_raw and |V+| / n extrapolated from
    the measured scales (1.735 / 1.872 / 1.912 / 1.940 at 16 / 20 /
    22 / 24; |V+| / n 0.715 / 0.616 / 0.571 / 0.529)."""
    n = 1 << scale
    m_raw = n * edgefactor
    md = int(m_raw * directed_per_raw)
    n_plus = int(n * nonisolated_frac)
    m_loc, md_loc, n_loc = m_raw // world, md // world, n // world
    GB = 1e9
    stages = {
        # edges (8 B) + 2 keys per edge, CUB double buffer + temp (~1 more buffer)
        "generate+local_build": (8 * m_loc + 3 * 8 * 2 * m_loc) / GB,
        # received keys + sort double buffer + temp; local CSR
        "route+merge": (3 * 8 * md_loc + 4 * md_loc + 8 * n_loc) / GB,
        # root: whole CSR (int32 cols, int64 row starts, int32 degrees) + rb_rcm workspace (~20 n-word arrays,
        # 2 n-entry uint64 key buffers, 2 n-entry int64 scans) + its own block
        "rcm_on_root": (4 * md + 12 * n + 20 * 4 * n + 4 * 8 * n + 4 * md_loc) / GB,
        # relabel keys + routed keys + sort buffers; the new block
        "relabel": (8 * md_loc * 4 + 4 * md_loc) / GB,
        # traversal: rows + transpose slice (int32 each), row records (16 B per local and per global vertex:
        # vinfo / td_vinfo), hot pairs, degrees, parents, local bitmaps, 3 global frontier bitmaps + summaries,
        # hub queues (<= td_m / 32 entries of 16 + 4 B, twice)
        "traversal": (2 * 4 * md_loc + 16 * n_loc + 16 * n_plus + 8 * n_loc + 8 * n_loc + 8 * n_loc
                      + 3 * (n_plus / 8 + n_plus / 32) + 2 * 20 * (md_loc / 32)) / GB,
    }
    return {"scale": scale, "world": world, "n": n, "m_raw": m_raw, "m_directed_est": md, "hbm_gb": hbm_gb,
            "stages_gb": {k: round(v, 2) for k, v in stages.items()},
            "peak_gb": round(max(stages.values()), 2), "fits": max(stages.values()) < hbm_gb}
