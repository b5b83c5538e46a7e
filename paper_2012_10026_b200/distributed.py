"""1D vertex-block partitioned BFS over P GPUs.

One process per GPU (``torch.distributed``, NCCL).  The RCM graph is built
replicated on every rank (RCM does not shard: SURVEY §8(e)); each rank then
keeps

* the CSR rows of its owned vertex block ``[lo, hi)`` (global column ids) --
  what its bottom-up steps scan, and
* the block's *transpose slice*: for every global vertex u, the owned vertices
  adjacent to u -- what its top-down steps expand, so a rank claims only
  vertices it owns and no second exchange is needed.

Block boundaries are aligned to 8192 vertices (whole 256-word bitmap tiles)
and balanced by edge count (RCM ids ascend with degree, so equal-vertex blocks
would be badly edge-imbalanced).

Per level every rank runs its local step (one kernel launch), then the ranks
all-reduce the counters {n_next, deg_next, scanned} (+ max degree) that drive
``update_traversal_policy`` and all-gather their next-frontier bitmap slices
into the global bitmap the next level reads (n/8 bytes in total).  The level
loop is the reference's (engine.py:534-598) with n = g.n.

``PartitionedBfs`` is the exchange/policy driver; the local step is pluggable
(``GpuLocalLevel`` here; the CPU tests plug in a numpy step over gloo).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

ALIGN = 8192  # vertices per partition-boundary unit (256 bitmap words)


def partition_bounds(row_starts: np.ndarray, n_dev: int, world: int, align: int = ALIGN) -> list[int]:
    """Edge-balanced split of [0, n_dev) into ``world`` blocks.

    Weight of a vertex = degree + 1; boundaries are multiples of ``align``
    (the last is n_dev), non-decreasing (a rank may own an empty block)."""
    rs = np.asarray(row_starts[: n_dev + 1], dtype=np.int64)
    weight = rs + np.arange(n_dev + 1, dtype=np.int64)  # cumulative (deg + 1)
    total = int(weight[-1])
    bounds = [0]
    for r in range(1, world):
        target = total * r // world
        v = int(np.searchsorted(weight, target, side="left"))
        v = (v // align) * align
        v = min(max(v, bounds[-1]), n_dev)
        bounds.append(v)
    bounds.append(n_dev)
    return bounds


def words_for(n_vertices: int, tile: int = ALIGN) -> int:
    """uint32 words of a bitmap over n vertices, padded like the device engine."""
    return ((n_vertices + tile - 1) // tile) * (tile // 32)


@dataclass
class DistRecord:
    level: int
    direction: int  # 0 TD, 1 BU
    n_f: int
    m_f: int
    m_u: int
    scanned: int


class PartitionedBfs:
    """Level-synchronous driver: local step + counter all-reduce + frontier all-gather.

    ``local`` must provide ``reset(source)``, ``level(L, direction, hubs,
    glob_words, glob_nz) -> (counters[4] int64 (n_next, deg_next, maxdeg,
    scanned), next_local_words)``, ``make_nz(glob_words)`` and
    ``zeros(n, dtype)``; tensors live on ``local.device``."""

    def __init__(self, local, bounds: list[int], rank: int, world: int, n_policy: int, m_directed: int,
                 alpha: int = 64, beta: int = 8, hybrid: bool = True, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.local = local
        self.bounds = bounds
        self.rank, self.world = rank, world
        self.n_policy, self.m_directed = n_policy, m_directed
        self.alpha, self.beta, self.hybrid = alpha, beta, hybrid
        self.group = group
        n_glob = bounds[-1]
        self.n_words_glob = words_for(n_glob)
        # gloo has no CUDA collectives: stage through host memory (CPU tests / one-GPU runs)
        self.stage = dist.get_backend(group) == "gloo" and self.local.device.type == "cuda"
        # rank r's slice = global words [lo_r / 32, lo_r / 32 + ceil((hi_r - lo_r) / 32)) (lo_r % 32 == 0)
        assert all(b % 32 == 0 for b in bounds[:-1])
        self.slice_words = [(bounds[r + 1] - bounds[r] + 31) // 32 for r in range(world)]
        self.send_words = max(max(self.slice_words), 32)

    # -- exchange ---------------------------------------------------------
    def _allgather_frontier(self, next_local):
        torch = self.torch
        dev = self.local.device
        send = torch.zeros(self.send_words, dtype=torch.int32, device=dev)
        k = self.slice_words[self.rank]
        if k:
            send[:k] = next_local[:k]
        if self.stage:
            send_h = send.cpu()
            recv_h = torch.empty(self.world * self.send_words, dtype=torch.int32)
            self.dist.all_gather_into_tensor(recv_h, send_h, group=self.group)
            recv = recv_h.to(dev)
        else:
            recv = torch.empty(self.world * self.send_words, dtype=torch.int32, device=dev)
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
        recv = recv.view(self.world, self.send_words)
        glob = torch.zeros(self.n_words_glob, dtype=torch.int32, device=dev)
        for r in range(self.world):
            kw = self.slice_words[r]
            if kw:
                w0 = self.bounds[r] // 32
                glob[w0 : w0 + kw] = recv[r, :kw]
        return glob

    def _allreduce(self, counters):
        torch = self.torch
        dev = self.local.device
        if self.stage:
            dev = torch.device("cpu")
        s = torch.tensor([counters[0], counters[1], counters[3]], dtype=torch.int64, device=dev)
        m = torch.tensor([counters[2]], dtype=torch.int64, device=dev)
        self.dist.all_reduce(s, op=self.dist.ReduceOp.SUM, group=self.group)
        self.dist.all_reduce(m, op=self.dist.ReduceOp.MAX, group=self.group)
        s = s.cpu().numpy()
        return int(s[0]), int(s[1]), int(m.item()), int(s[2])

    # -- the level loop (engine.py:534-598) --------------------------------
    def run(self, source: int, deg_source: int) -> list[DistRecord]:
        torch = self.torch
        self.local.reset(source)
        glob = torch.zeros(self.n_words_glob, dtype=torch.int32, device=self.local.device)
        glob[source >> 5] = int(np.int32(np.uint32(1 << (source & 31))))
        nz = self.local.make_nz(glob)
        nf, mf, mu = 1, deg_source, self.m_directed - deg_source
        direction, hubs = 0, deg_source > 32
        records: list[DistRecord] = []
        level = 0
        while nf > 0:
            cnt, nxt = self.local.level(level, direction, hubs, glob, nz)
            n_next, deg_next, maxdeg, scanned = self._allreduce(cnt)
            records.append(DistRecord(level, direction, nf, mf, mu, scanned))
            mu -= deg_next
            mf = deg_next
            nf = n_next
            if self.hybrid:  # update_traversal_policy (engine.py:215-228), n = g.n
                if direction == 0:
                    direction = 1 if mf > mu / self.alpha else 0
                else:
                    direction = 0 if nf < self.n_policy / self.beta else 1
            hubs = maxdeg > 32
            if nf > 0:
                glob = self._allgather_frontier(nxt)
                nz = self.local.make_nz(glob)
            level += 1
        return records


class GpuLocalLevel:
    """The local step of one rank: an rb_bfs engine created with a partition."""

    def __init__(self, g, bounds: list[int], rank: int, alpha: int, beta: int, hybrid: bool = True,
                 record_levels: bool = False, rows=None):
        """``g``: the whole RCM graph (every rank slices its block), or None
        with ``rows`` = this rank's block (sharded.LocalRows, new ids) and
        ``g`` replaced by (n, m_directed) for the policy."""
        torch = _lib.require_cuda()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        L = _lib.lib()
        lo, hi = bounds[rank], bounds[rank + 1]
        self.lo, self.hi = lo, hi
        n_glob = bounds[-1]
        n_local = hi - lo
        self.n_local = n_local
        s = _lib.stream_ptr()
        self._empty = torch.zeros(32, dtype=torch.int32, device=self.device)
        self.n_words_local = 0
        if rows is None:
            n_policy, m_directed = g.n, g.m_directed
        else:
            n_policy, m_directed = g
        if n_local == 0:
            self.h = None
            return
        if rows is None:
            rs, col, deg = g.device_arrays()
            e0, e1 = int(rs[lo].item()), int(rs[hi].item())
            self.rs_local = (rs[lo : hi + 1] - e0).contiguous()
            self.col_local = col[e0:e1]
            self.deg_local = deg[lo:hi].contiguous()
        else:
            assert (rows.lo, rows.hi) == (lo, hi), "rows do not match the partition bounds"
            self.rs_local, self.col_local, self.deg_local = rows.rs, rows.col, rows.deg
            e0, e1 = 0, rows.m_local
        m_local = e1 - e0
        # transpose slice: owned neighbours of every global vertex
        ws_bytes = L.rb_transpose_workspace_bytes(m_local, n_glob)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.device)
        self.td_rs = torch.empty(n_glob + 1, dtype=torch.int64, device=self.device)
        self.td_col = torch.empty(max(m_local, 1), dtype=torch.int32, device=self.device)
        _lib.check(L.rb_transpose_rows(_lib.ptr(self.rs_local), _lib.ptr(self.col_local), n_local, lo, m_local,
                                       n_glob, _lib.ptr(ws), ws_bytes, _lib.ptr(self.td_rs), _lib.ptr(self.td_col), s),
                   "rb_transpose_rows")
        del ws
        # isolated vertices inside the owned block are premarked visited
        nw = (n_local + 31) // 32
        flags = torch.zeros(nw * 32, dtype=torch.int64, device=self.device)
        flags[:n_local] = (self.deg_local == 0).to(torch.int64)
        words = (flags.view(nw, 32) << torch.arange(32, device=self.device, dtype=torch.int64)).sum(dim=1)
        self.iso = torch.where(words >= (1 << 31), words - (1 << 32), words).to(torch.int32)
        prm = _lib.BfsParamsC(alpha, beta, int(hybrid), 1, n_policy, m_directed, int(record_levels), 0)
        part = _lib.PartitionC(lo, n_glob, _lib.ptr(self.td_rs).value, _lib.ptr(self.td_col).value)
        self.h = ctypes.c_void_p(0)
        _lib.check(L.rb_bfs_create_part(_lib.ptr(self.rs_local), _lib.ptr(self.col_local), _lib.ptr(self.col_local),
                                        _lib.ptr(self.deg_local), n_local, _lib.ptr(self.iso), ctypes.byref(prm),
                                        ctypes.byref(part), ctypes.byref(self.h)), "rb_bfs_create_part")
        nwl, nwg = ctypes.c_int64(0), ctypes.c_int64(0)
        L.rb_bfs_words(self.h, ctypes.byref(nwl), ctypes.byref(nwg))
        self.n_words_local = nwl.value

    def close(self):
        if self.h:
            _lib.lib().rb_bfs_destroy(self.h)
            self.h = None

    def reset(self, source: int):
        if self.h:
            _lib.check(_lib.lib().rb_bfs_reset_part(self.h, int(source), _lib.stream_ptr()), "rb_bfs_reset_part")

    def make_nz(self, glob):
        nz = self.torch.empty(glob.numel(), dtype=self.torch.uint8, device=self.device)  # one byte per word
        _lib.check(_lib.lib().rb_make_nz(_lib.ptr(glob), glob.numel(), _lib.ptr(nz), _lib.stream_ptr()), "rb_make_nz")
        return nz

    def level(self, L: int, direction: int, hubs: bool, glob, nz):
        if not self.h:
            return np.zeros(4, np.int64), self._empty
        cnt = np.zeros(4, np.int64)
        nxt = ctypes.c_void_p(0)
        _lib.check(_lib.lib().rb_bfs_dist_level(self.h, L, direction, int(hubs), _lib.ptr(glob), _lib.ptr(nz),
                                                ctypes.byref(nxt), cnt.ctypes.data_as(ctypes.c_void_p),
                                                _lib.stream_ptr()), "rb_bfs_dist_level")
        from .engine import _ptr_view

        return cnt, _ptr_view(nxt.value, self.n_words_local)

    def parents(self):
        """int32 CUDA tensor view of the owned block's parents (global ids)."""
        from .engine import _ptr_view

        if not self.h:
            return self.torch.empty(0, dtype=self.torch.int32, device=self.device)
        return _ptr_view(_lib.lib().rb_bfs_parent_ptr(self.h), self.n_local)

    def levels(self):
        from .engine import _ptr_view

        if not self.h:
            return self.torch.empty(0, dtype=self.torch.int32, device=self.device)
        return _ptr_view(_lib.lib().rb_bfs_level_ptr(self.h), self.n_local)


# ---------------------------------------------------------------------------
# The exchange on the device: one persistent launch per rank per root
# (rb_bfs.cu bfs_dist).  Each rank stores its next-frontier words and level
# counters straight into every rank's buffers (CUDA IPC mappings over NVLink)
# and meets the others at a system-scope barrier -- no host round trip and no
# NCCL call per level.  On one GPU the ranks run as ONE cooperative launch over
# all their data (bfs_dist_emu), the way the profiling guide asks multi-rank
# kernels that wait on each other to be tested with fewer GPUs than ranks.


class DevicePartition:
    """One rank's engine (owned rows + transpose slice, GpuLocalLevel) plus its
    exchange buffers: three global frontier bitmaps + summaries, the counter
    slots and the cross-rank barrier counter, in one IPC-exportable block."""

    def __init__(self, g, bounds: list[int], rank: int, world: int, alpha: int = 64, beta: int = 8,
                 hybrid: bool = True, record_levels: bool = False, rows=None):
        if any(bounds[r + 1] <= bounds[r] for r in range(world)):
            raise ValueError(f"every rank needs a non-empty vertex block, got bounds {bounds}")
        self.local = GpuLocalLevel(g, bounds, rank, alpha, beta, hybrid, record_levels, rows=rows)
        self.rank, self.world = rank, world
        self.bounds = bounds
        self.g = g
        _lib.check(_lib.lib().rb_bfs_xchg_alloc(self.local.h, world, rank), "rb_bfs_xchg_alloc")

    @property
    def h(self):
        return self.local.h

    def handle(self) -> bytes:
        L = _lib.lib()
        buf = (ctypes.c_char * int(L.rb_bfs_xchg_handle_bytes()))()
        _lib.check(L.rb_bfs_xchg_handle(self.h, buf), "rb_bfs_xchg_handle")
        return bytes(buf)

    def open(self, handles: list[bytes]) -> None:
        blob = b"".join(handles)
        _lib.check(_lib.lib().rb_bfs_xchg_open(self.h, ctypes.c_char_p(blob)), "rb_bfs_xchg_open")

    def reset(self, source: int, deg_source: int) -> None:
        _lib.check(_lib.lib().rb_bfs_dist_reset(self.h, int(source), int(deg_source), _lib.stream_ptr()),
                   "rb_bfs_dist_reset")

    def traverse(self) -> None:
        _lib.check(_lib.lib().rb_bfs_dist_traverse(self.h, _lib.stream_ptr()), "rb_bfs_dist_traverse")

    def results(self, timed: bool = True):
        """(records [DistRecord], executed directions, device seconds) of the
        last traversal; the records are rank 0's (identical on every rank).
        ``timed=False``: the engine did not record the launch (emulated ranks > 0)."""
        recs = (_lib.LevelRecordC * 4096)()
        nrec = ctypes.c_int64(0)
        el = ctypes.c_double(0.0)
        _lib.check(_lib.lib().rb_bfs_dist_results(self.h, recs, len(recs), ctypes.byref(nrec),
                                                  ctypes.byref(el) if timed else None, _lib.stream_ptr()),
                   "rb_bfs_dist_results")
        out = [DistRecord(int(r.level), int(r.direction), int(r.n_f), int(r.m_f), int(r.m_u), int(r.scanned_edges))
               for r in recs[: nrec.value]]
        return out, [int(r.reserved) for r in recs[: nrec.value]], el.value

    def close(self) -> None:
        self.local.close()


def connect_emulated(parts: list[DevicePartition]) -> None:
    """One process, one GPU: every rank's peers are the other engines' buffers."""
    arr = (ctypes.c_void_p * len(parts))(*[p.h.value for p in parts])
    _lib.check(_lib.lib().rb_bfs_xchg_connect_local(arr, len(parts)), "rb_bfs_xchg_connect_local")


def run_emulated(parts: list[DevicePartition], source: int, deg_source: int):
    """All ranks' traversal of one root in ONE cooperative launch on this GPU;
    returns rank 0's (records, executed directions, device seconds)."""
    for p in parts:
        p.reset(source, deg_source)
    arr = (ctypes.c_void_p * len(parts))(*[p.h.value for p in parts])
    _lib.check(_lib.lib().rb_bfs_dist_traverse_emu(arr, len(parts), _lib.stream_ptr()), "rb_bfs_dist_traverse_emu")
    res = parts[0].results()
    for p in parts[1:]:
        p.results(timed=False)  # (clears the launched state of every engine)
    return res


class DeviceExchangeBfs:
    """Multi-process driver (one rank per GPU): IPC handles are exchanged once
    through torch.distributed, then every root is reset + ONE launch per rank."""

    def __init__(self, g, bounds: list[int], rank: int, world: int, alpha: int = 64, beta: int = 8,
                 hybrid: bool = True, record_levels: bool = False, group=None, rows=None):
        import torch.distributed as dist

        self.part = DevicePartition(g, bounds, rank, world, alpha, beta, hybrid, record_levels, rows=rows)
        handles = [None] * world
        dist.all_gather_object(handles, self.part.handle(), group=group)
        self.part.open(handles)
        dist.barrier(group=group)

    @property
    def local(self):
        return self.part.local

    def run(self, source: int, deg_source: int):
        self.part.reset(source, deg_source)
        self.part.traverse()
        recs, _, _ = self.part.results()
        return recs

    def elapsed(self) -> float:
        el = ctypes.c_double(0.0)
        _lib.check(_lib.lib().rb_bfs_elapsed(self.part.h, ctypes.byref(el)), "rb_bfs_elapsed")
        return el.value

    def close(self):
        self.part.close()
