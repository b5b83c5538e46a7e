"""Direction-optimizing BFS engine on B200 (reference engine.py:1-639).

Same public surface as the reference (``BfsParams``, ``BfsEngine``,
``bfs_run``, the step functions, ``update_traversal_policy``...), but every
traversal runs on the device through the C ABI (include/rcmbfs_b200.h):

* ``BfsEngine.run`` = reset (untimed, engine.py:526-532) + ONE cooperative
  persistent kernel for the whole level loop (engine.py:534-598) + copy-out.
  The per-level direction policy runs on device with exactly
  ``update_traversal_policy``'s arithmetic (n = g.n including isolated).
* Isolated vertices beyond the last non-isolated id are dropped from the
  device state (after RCM they are the tail [|V+|, n)); isolated vertices
  inside the range are premarked visited (engine.py:432-437).
* Modes: ``hybrid`` (the fast path) scans bottom-up rows from their end (RCM
  ids ascend with degree) and executes each level the cheaper way, keeping
  the policy's labels; its levels, directions and n_f / m_f / m_u equal the
  reference's.  The paper's modes run every level as labelled and scan in
  the reference's order -- ``hybrid_balanced`` the ascending rows (bu_steal),
  ``hybrid_reduced`` the descending-degree adjacency ``g_desc`` (Alg. 6
  bu_reduced) -- so their LevelRecords match the reference field for field:
  scanned_edges, pass1_hits, live_vertices (partition.py shrink rule over
  get_partitions(n, partition_factor, threads)) and claimed.  ``level_sync``
  and ``sequential`` are top-down only.  Parents may differ from the CPU
  reference's (any valid BFS tree).

There is no CPU fallback: constructing an engine without CUDA raises.
"""

from __future__ import annotations

import csv
import ctypes
import mmap
import os
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bitmap import Bitmap
from .graph import CsrGraph

__all__ = [
    "TOP_DOWN", "BOTTOM_UP", "MODES", "BfsParams", "Frontier", "StepStats", "LevelRecord", "BfsResult",
    "PolicyCounters", "update_traversal_policy", "default_partition_factor", "top_down_step",
    "top_down_step_balanced", "bottom_up_step", "bottom_up_step_balanced", "bottom_up_step_reduced",
    "bfs_sequential", "bfs_run", "BfsEngine", "write_level_trace",
]

TOP_DOWN = "top_down"
BOTTOM_UP = "bottom_up"
MODES = ("sequential", "level_sync", "hybrid", "hybrid_balanced", "hybrid_reduced")
_PARTITIONED_MODES = ("hybrid_balanced", "hybrid_reduced")


def default_partition_factor(n: int) -> int:
    """engine.py:70-72."""
    return 10 if n < (1 << 26) else 20


@dataclass
class BfsParams:
    """Traversal configuration (engine.py:75-103), same validation."""

    alpha: int = 64
    beta: int = 8
    partition_factor: int = 20
    threads: int = 1
    mode: str = "hybrid"

    def __post_init__(self):
        if not 1 <= self.alpha <= 128:
            raise ValueError(f"alpha must be in [1, 128], got {self.alpha}")
        if not 1 <= self.beta <= 32:
            raise ValueError(f"beta must be in [1, 32], got {self.beta}")
        if self.partition_factor < 1:
            raise ValueError(f"partition_factor must be >= 1, got {self.partition_factor}")
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")


@dataclass
class Frontier:
    """One level's vertex set in queue and/or bitmap form (engine.py:106-151)."""

    n: int
    queue: np.ndarray | None = None
    bits: Bitmap | None = None
    active: str = "queue"

    @classmethod
    def from_queue(cls, n: int, queue: np.ndarray) -> "Frontier":
        return cls(n=n, queue=np.ascontiguousarray(queue, dtype=np.uint32), active="queue")

    @classmethod
    def from_bitmap(cls, bits: Bitmap) -> "Frontier":
        return cls(n=bits.n_bits, bits=bits, active="bitmap")

    @property
    def count(self) -> int:
        if self.queue is not None:
            return int(self.queue.size)
        return self.bits.count()

    def indices(self) -> np.ndarray:
        if self.queue is not None:
            return self.queue
        return self.bits.to_indices()

    def to_queue_form(self) -> "Frontier":
        if self.queue is not None:
            return self
        return Frontier(n=self.n, queue=self.bits.to_indices(), bits=self.bits, active="queue")

    def to_bitmap_form(self) -> "Frontier":
        if self.bits is not None:
            return self
        return Frontier(n=self.n, queue=self.queue, bits=Bitmap.from_indices(self.n, self.queue), active="bitmap")


@dataclass
class StepStats:
    n_next: int
    deg_next: int
    scanned_edges: int
    per_thread_edges: np.ndarray
    pass1_hits: int | None = None
    claimed: int | None = None


@dataclass
class LevelRecord:
    """Per-level trace entry (engine.py:166-180); wall_time is device time."""

    level: int
    direction: str
    n_f: int
    m_f: int
    m_u: int
    scanned_edges: int
    wall_time: float
    per_thread_edges: np.ndarray | None = None
    pass1_hits: int | None = None
    live_vertices: int | None = None
    claimed: int | None = None
    queue_time: float = 0.0  # device seconds of this level spent rebuilding top-down queues
    # how the device ran the level: the policy's label is `direction`; a level
    # labelled bottom-up with few frontier edges may run top-down
    executed_direction: str | None = None


@dataclass
class BfsResult:
    source: int
    n: int
    predecessor: np.ndarray
    levels: list
    elapsed_time: float
    traversed_edges: int
    mode: str

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    @property
    def n_reached(self) -> int:
        return int(np.count_nonzero(self.predecessor >= 0))


@dataclass
class PolicyCounters:
    direction: str
    m_f: int
    m_u: int
    n_f: int
    n: int


def update_traversal_policy(counters: PolicyCounters, params: BfsParams) -> str:
    """engine.py:215-228 (the device kernel evaluates the same expression)."""
    if counters.direction == TOP_DOWN:
        if counters.m_f > counters.m_u / params.alpha:
            return BOTTOM_UP
        return TOP_DOWN
    if counters.n_f < counters.n / params.beta:
        return TOP_DOWN
    return BOTTOM_UP


def _split_even(total: int, parts: int) -> np.ndarray:
    """Device work reported as `parts` equal shares (per_thread_edges field)."""
    return np.array([total * (k + 1) // parts - total * k // parts for k in range(parts)], dtype=np.int64)


# ---------------------------------------------------------------------------
# device engine handle


class _DeviceBfs:
    """Owns one rb_bfs handle: graph views + device traversal state."""

    def __init__(self, g: CsrGraph, *, hybrid: bool, alpha: int, beta: int, g_bu: CsrGraph | None,
                 bu_reverse: bool, trim_isolated: bool, record_levels: bool = False):
        torch = _lib.require_cuda()
        self.torch = torch
        self.record_levels = record_levels
        L = _lib.lib()
        self.g = g
        rs, col, deg = g.device_arrays()
        self._keep = [rs, col, deg]
        n = g.n
        if trim_isolated:
            nz = torch.nonzero(deg > 0)
            n_dev = int(nz.max().item()) + 1 if nz.numel() else 0
        else:
            n_dev = n
        self.n_dev = n_dev
        self.h = ctypes.c_void_p(0)
        if n_dev == 0:
            return
        iso = None
        if trim_isolated:
            nw = (n_dev + 31) // 32
            flags = torch.zeros(nw * 32, dtype=torch.int64, device="cuda")
            flags[:n_dev] = (deg[:n_dev] == 0).to(torch.int64)
            shifts = torch.arange(32, device="cuda", dtype=torch.int64)
            words = (flags.view(nw, 32) << shifts).sum(dim=1)
            iso = torch.where(words >= (1 << 31), words - (1 << 32), words).to(torch.int32)  # uint32 bit pattern
            self._keep.append(iso)
        col_bu = col
        if g_bu is not None:
            col_bu = g_bu.device_arrays()[1]
            self._keep.append(col_bu)
        prm = _lib.BfsParamsC(alpha, beta, int(hybrid), int(bu_reverse), n, g.m_directed, int(record_levels), 0)
        # rb_bfs_create reads deg / iso from its own (legacy default) stream:
        # the torch work above must have landed, whatever stream it ran on
        torch.cuda.current_stream().synchronize()
        _lib.check(
            L.rb_bfs_create(_lib.ptr(rs), _lib.ptr(col), _lib.ptr(col_bu), _lib.ptr(deg), n_dev,
                            _lib.ptr(iso) if iso is not None else None, ctypes.byref(prm), ctypes.byref(self.h)),
            "rb_bfs_create",
        )
        self.pinned = torch.empty(n_dev, dtype=torch.int32, pin_memory=True)
        self._state = None  # pinned launch state + records of the async result path
        self._recs = (_lib.LevelRecordC * 256)()

    def close(self):
        if self.h:
            _lib.lib().rb_bfs_destroy(self.h)
            self.h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def traverse(self, source: int):
        """Reset + timed traversal; returns device seconds."""
        L = _lib.lib()
        s = _lib.stream_ptr()
        _lib.check(L.rb_bfs_reset(self.h, int(source), s), "rb_bfs_reset")
        _lib.check(L.rb_bfs_traverse(self.h, s), "rb_bfs_traverse")

    def results(self, want_parent=True, level_out=None, parent_host=None):
        """Drain the traversal; copy parents (to ``parent_host`` numpy int32
        array if given, else the pinned buffer) and return (records, seconds)."""
        L = _lib.lib()
        nrec = ctypes.c_int64(0)
        if parent_host is not None:
            pdst = ctypes.c_void_p(parent_host.ctypes.data)
        elif want_parent:
            pdst = _lib.ptr(self.pinned)
        else:
            pdst = None
        _lib.check(
            L.rb_bfs_results(self.h, pdst, _lib.ptr(level_out) if level_out is not None else None, self._recs,
                             len(self._recs), ctypes.byref(nrec), _lib.stream_ptr()),
            "rb_bfs_results",
        )
        if nrec.value > len(self._recs):  # very deep traversal: records are kept host-side until reset
            self._recs = (_lib.LevelRecordC * nrec.value)()
            _lib.check(L.rb_bfs_results(self.h, None, None, self._recs, len(self._recs), ctypes.byref(nrec),
                                        _lib.stream_ptr()), "rb_bfs_results")
        el = ctypes.c_double(0.0)
        _lib.check(L.rb_bfs_elapsed(self.h, ctypes.byref(el)), "rb_bfs_elapsed")  # all launches of the traversal
        return self._recs[: nrec.value], el.value

    def run_to_host(self, source: int, n: int, chunks: int = 0):
        """BfsEngine.run's result path: reset + launch, then -- all enqueued
        behind the traversal -- the launch state, the level records and the
        parents [0, n_dev).  Large results go straight into the fresh result
        array (a pooled hugepage mapping page-locked once, so one DMA and no
        host copy); small ones through the pinned staging buffer in chunks,
        each landed chunk copied out while the next is in flight.  The
        isolated tail is filled with -1 while the GPU works.  Returns
        (predecessor, records, seconds)."""
        torch = self.torch
        L = _lib.lib()
        s = _lib.stream_ptr()
        self.traverse(source)
        if self._state is None:
            self._state = torch.empty(int(L.rb_bfs_state_bytes()) // 8, dtype=torch.int64, pin_memory=True)
            self._recs_pin = torch.empty(_REC_FAST * ctypes.sizeof(_lib.LevelRecordC) // 8, dtype=torch.int64,
                                         pin_memory=True)
        n_dev = self.n_dev
        pred, registered = fresh_int32(n, want_registered=True)
        if registered:
            # the result array is page-locked (pooled, registered once): the
            # parents are DMA'd straight into it in one copy, no staging hop
            chunks = 1
            dst = pred.ctypes.data
        else:
            # 8 pieces by default (the ABI accepts 1..32): measured best at s22 and s26
            # (1 / 2 / 4 / 8 -> 128 / 146 / 156 / 159 e2e GTEPS at s22; 16 / 32 lose)
            chunks = chunks or int(os.environ.get("RB_E2E_CHUNKS", "0")) or 8
            if not 1 <= chunks <= _MAX_CHUNKS:
                raise ValueError(f"result chunks must be in [1, {_MAX_CHUNKS}], got {chunks}")
            dst = _lib.ptr(self.pinned)
        _lib.check(L.rb_bfs_results_async(self.h, _lib.ptr(self._state), _lib.ptr(self._recs_pin), _REC_FAST,
                                          dst, chunks, s), "rb_bfs_results_async")
        pt = torch.from_numpy(pred)
        if n - n_dev >= _FILL_STREAM_MIN:
            # a big isolated tail: streaming stores from a few threads while the GPU works (a cached
            # fill takes host memory bandwidth from the parents' DMA)
            _lib.check(L.rb_host_fill_i32(ctypes.c_void_p(pred.ctypes.data + 4 * n_dev), n - n_dev, -1, _FILL_THREADS),
                       "rb_host_fill_i32")
        elif n > n_dev:  # small: torch's resident thread pool (spawning fill threads would cost more)
            pt[n_dev:].fill_(-1)
        _lib.check(L.rb_bfs_wait(self.h, -1), "rb_bfs_wait")
        nrec = ctypes.c_int64(0)
        done = L.rb_bfs_complete(self.h, _lib.ptr(self._state), _lib.ptr(self._recs_pin), _REC_FAST,
                                 ctypes.byref(nrec))
        if done == 0:
            recs = (_lib.LevelRecordC * nrec.value).from_buffer_copy(
                self._recs_pin.numpy().tobytes()[: nrec.value * ctypes.sizeof(_lib.LevelRecordC)])
            step = -(-n_dev // chunks)
            for i in range(chunks):
                a, b = i * step, min((i + 1) * step, n_dev)
                _lib.check(L.rb_bfs_wait(self.h, i), "rb_bfs_wait")
                if b > a and not registered:
                    pt[a:b].copy_(self.pinned[a:b])
            el = ctypes.c_double(0.0)
            _lib.check(L.rb_bfs_elapsed(self.h, ctypes.byref(el)), "rb_bfs_elapsed")
            return pred, recs, el.value
        # continuation launches (very deep traversal): drain, then copy again
        torch.cuda.synchronize()
        recs, el = self.results(want_parent=False)
        self.parents_to_host(pred, chunks=chunks)
        return pred, recs, el

    def parents_to_host(self, out: np.ndarray, chunks: int = 4):
        """Copy the parents [0, n_dev) into ``out`` (int32 numpy, length >= n_dev;
        the tail is set to -1): pinned-buffer DMA in chunks, each chunk's
        multi-threaded host copy overlapping the next chunk's transfer."""
        torch = self.torch
        n_dev = self.n_dev
        dev = _ptr_view(_lib.lib().rb_bfs_parent_ptr(self.h), n_dev)
        pt = torch.from_numpy(out)
        step = -(-n_dev // chunks)
        evs = []
        for a in range(0, n_dev, step):
            b = min(a + step, n_dev)
            self.pinned[a:b].copy_(dev[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            evs.append((a, b, ev))
        pt[n_dev:].fill_(-1)
        for a, b, ev in evs:
            ev.synchronize()
            pt[a:b].copy_(self.pinned[a:b])

    def level_tensor(self):
        """Device int32 level array over [0, n_dev) (valid after results())."""
        ptr = _lib.lib().rb_bfs_level_ptr(self.h)
        return ptr


_MAX_CHUNKS = 32  # kMaxChunks of rb_bfs.cu (rb_bfs_results_async)
_FILL_THREADS = int(os.environ.get("RB_FILL_THREADS", "0")) or min(8, os.cpu_count() or 1)
_FILL_STREAM_MIN = 8 << 20  # entries (32 MB) from which the tail fill uses rb_host_fill_i32
_REC_FAST = 64  # level records fetched by the async result path (deeper: drained)


class _Holder:
    """Exports one pooled mapping through the buffer protocol; every array
    view of it keeps the holder alive, and the mapping returns to the pool
    only when the last view is gone."""

    __slots__ = ("mm", "__weakref__")

    def __init__(self, mm):
        self.mm = mm

    def __buffer__(self, flags):
        return memoryview(self.mm)

    def __release_buffer__(self, view):
        view.release()


class _ResultPool:
    """Anonymous hugepage mappings for result arrays, reused once their
    previous owner is garbage: a returned predecessor array is always a new
    object that nobody else references, but its pages are already faulted in
    (first touch of a 100+ MB array costs more than the copy into it)."""

    def __init__(self, keep: int = 2):
        self.keep = keep
        self.free: dict[int, list] = {}
        self.lock = threading.Lock()
        self.registered: set[int] = set()  # id() of mappings page-locked with cudaHostRegister
        self.seen: set[int] = set()  # sizes requested so far

    def get(self, nbytes: int, register: bool = False):
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                return lst.pop()
            first = nbytes not in self.seen
            self.seen.add(nbytes)
        if first and self.keep > 1:
            # a caller that keeps the previous result while asking for the next
            # (res = eng.run(...) in a loop) needs two: make the spare now, not
            # in the middle of the loop (a fresh mapping + page lock costs ~40 ms)
            self.put(self._new(nbytes, register))
        return self._new(nbytes, register)

    def _new(self, nbytes: int, register: bool):
        m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if hasattr(m, "madvise") and hasattr(mmap, "MADV_HUGEPAGE"):
            m.madvise(mmap.MADV_HUGEPAGE)
        if register:
            # page-locked once for the life of the mapping (pool entries are never
            # unmapped), so the device copies straight into the result array
            import torch

            addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
            if int(torch.cuda.cudart().cudaHostRegister(addr, nbytes, 0)) == 0:
                self.registered.add(id(m))
        return m

    def put(self, m):
        with self.lock:
            lst = self.free.setdefault(len(m), [])
            if len(lst) < self.keep:
                lst.append(m)
                return
            registered = id(m) in self.registered
            self.registered.discard(id(m))
        if registered:  # dropped from the pool: unlock before the mapping goes away
            import torch

            torch.cuda.cudart().cudaHostUnregister(ctypes.addressof(ctypes.c_char.from_buffer(m)))


_POOL = _ResultPool()


def fresh_int32(n: int, want_registered: bool = False):
    """A new int32 array of n entries (contents undefined).  Up to 32 MB:
    np.empty (glibc reuses already-faulted heap pages).  Larger: a pooled
    hugepage mapping (see _ResultPool) -- first touch of fresh 4 KB pages
    runs at ~8 GB/s, a warm pooled buffer is written at ~50 GB/s; with
    ``want_registered`` the mapping is also page-locked (RB_E2E_REGISTER=0
    turns that off) and (array, registered) is returned."""
    if n < (8 << 20):
        a = np.empty(n, dtype=np.int32)
        return (a, False) if want_registered else a
    reg = want_registered and os.environ.get("RB_E2E_REGISTER", "1") != "0"
    m = _POOL.get(4 * n, register=reg)
    h = _Holder(m)
    weakref.finalize(h, _POOL.put, m)
    a = np.frombuffer(h, dtype=np.int32)
    return (a, id(m) in _POOL.registered) if want_registered else a


def _records_to_levels(recs, part=None) -> list:
    """Device records -> LevelRecords.  ``part`` = (n_partitions, live_fixed):
    the partitioned modes' bottom-up levels report ``claimed`` = every
    partition (each is claimed once per step, _kernels.py:176-293) and, for
    hybrid_balanced (bounds never shrink), ``live_vertices`` = live_fixed."""
    out = []
    for r in recs:
        bu = r.direction != 0
        claimed = part[0] if (part is not None and bu) else None
        live = int(r.live_vertices) if r.live_vertices >= 0 else None
        if part is not None and bu and part[1] is not None:
            live = part[1]
        out.append(
            LevelRecord(
                level=int(r.level), direction=TOP_DOWN if r.direction == 0 else BOTTOM_UP, n_f=int(r.n_f),
                m_f=int(r.m_f), m_u=int(r.m_u), scanned_edges=int(r.scanned_edges), wall_time=r.t_ns * 1e-9,
                per_thread_edges=np.array([int(r.scanned_edges)], dtype=np.int64), queue_time=r.t_queue_ns * 1e-9,
                executed_direction=TOP_DOWN if r.reserved == 0 else BOTTOM_UP,
                pass1_hits=int(r.pass1_hits) if r.pass1_hits >= 0 else None, live_vertices=live, claimed=claimed,
            )
        )
    return out


class BfsEngine:
    """Reusable traversal context (engine.py:478-604): device state per graph."""

    def __init__(self, g: CsrGraph, params: BfsParams, g_desc: CsrGraph | None = None, *,
                 record_levels: bool = False):
        """``record_levels`` (an extension, not in the reference) also keeps a
        per-vertex level array on the device (``level_device``); it costs one
        extra 4-byte write per reached vertex inside the traversal."""
        self.g = g
        self.params = params
        self.g_desc = g_desc
        if params.mode == "hybrid_reduced":
            if g_desc is None:
                raise ValueError(
                    "hybrid_reduced needs the descending-degree adjacency "
                    "variant (pass g_desc, e.g. degree_sort_adjacency(g))"
                )
            if g_desc.n != g.n or g_desc.m_directed != g.m_directed:
                raise ValueError("g_desc does not match g")
        self.ps = None
        self.pool = None  # device engine: no host worker pool
        hybrid = params.mode not in ("sequential", "level_sync")
        reduced = params.mode == "hybrid_reduced"
        partitioned = params.mode in _PARTITIONED_MODES
        # hybrid: bottom-up rows scanned from their end (RCM ids ascend with
        # degree) and each level executed the cheaper way.  The paper's modes
        # run exactly as labelled and scan in the reference's order (ascending
        # rows for hybrid_balanced, the descending-degree adjacency for
        # hybrid_reduced), so every LevelRecord field equals the reference's.
        self._dev = _DeviceBfs(
            g, hybrid=hybrid, alpha=params.alpha, beta=params.beta, g_bu=g_desc if reduced else None,
            bu_reverse=not partitioned, trim_isolated=True, record_levels=record_levels,
        )
        self._part = None
        if partitioned and g.n >= 1:
            from .partition import get_partitions

            self.ps = get_partitions(g.n, params.partition_factor, params.threads)  # engine.py:499-500
            flags = _lib.RB_PART_EXACT
            if reduced:
                flags |= _lib.RB_PART_COUNT_PASS1 | _lib.RB_PART_SHRINK
            if self._dev.h:
                st = np.ascontiguousarray(self.ps.starts, dtype=np.int64)
                _lib.check(_lib.lib().rb_bfs_set_partitions(self._dev.h, st.ctypes.data_as(ctypes.c_void_p),
                                                            st.size, g.n, flags), "rb_bfs_set_partitions")
            self._part = (self.ps.n_partitions, None if reduced else g.n)
        self._deg_host = g.degrees  # host copy (once per graph): the per-run isolated-source check

    @property
    def n_dev(self) -> int:
        return self._dev.n_dev

    def close(self) -> None:
        if self._dev is not None:
            self._dev.close()

    def __enter__(self) -> "BfsEngine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def _trivial(self, source: int) -> BfsResult:
        g = self.g
        pred = np.full(g.n, -1, dtype=np.int32)
        pred[source] = source
        rec = LevelRecord(level=0, direction=TOP_DOWN, n_f=1, m_f=0, m_u=g.m_directed, scanned_edges=0,
                          wall_time=0.0, per_thread_edges=np.zeros(1, np.int64))
        return BfsResult(source=source, n=g.n, predecessor=pred, levels=[rec], elapsed_time=0.0,
                         traversed_edges=0, mode=self.params.mode)

    def run(self, source: int) -> BfsResult:
        g = self.g
        if not 0 <= source < g.n:
            raise ValueError(f"source {source} out of range for n={g.n}")
        source = int(source)
        if source >= self._dev.n_dev or int(self._deg_host[source]) == 0:
            return self._trivial(source)
        pred, recs, elapsed = self._dev.run_to_host(source, g.n)
        levels = _records_to_levels(recs, self._part)
        traversed = sum(r.m_f for r in levels) // 2  # = sum deg[reached] // 2 (engine.py:599-600)
        return BfsResult(source=source, n=g.n, predecessor=pred, levels=levels, elapsed_time=elapsed,
                         traversed_edges=traversed, mode=self.params.mode)

    # ---- device-resident entry points (bench / parity tests) ------------
    def run_device(self, source: int, levels_out=None):
        """Traverse without copying parents to the host.  Returns
        (device seconds, LevelRecords).  If ``levels_out`` (int32 CUDA
        tensor of n_dev) is given, the level array is copied into it."""
        self._dev.traverse(int(source))
        recs, elapsed = self._dev.results(want_parent=False, level_out=levels_out)
        return elapsed, _records_to_levels(recs, self._part)

    def parent_device(self):
        """int32 CUDA tensor view of the engine's parent array [0, n_dev)."""
        return _ptr_view(_lib.lib().rb_bfs_parent_ptr(self._dev.h), self._dev.n_dev)

    def level_device(self):
        if not self._dev.record_levels:
            raise ValueError("engine created without record_levels=True")
        return _ptr_view(_lib.lib().rb_bfs_level_ptr(self._dev.h), self._dev.n_dev)


def _ptr_view(ptr: int, n: int):
    """Non-owning int32 CUDA tensor over an engine buffer."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": "<i4", "data": (int(ptr), False), "version": 3, "strides": None,
        }

    return torch.as_tensor(_Holder(), device="cuda")


def bfs_run(g: CsrGraph, source: int, params: BfsParams | None = None, g_desc: CsrGraph | None = None) -> BfsResult:
    """One-shot traversal (engine.py:607-617)."""
    if params is None:
        params = BfsParams()
    with BfsEngine(g, params, g_desc=g_desc) as eng:
        return eng.run(source)


def bfs_sequential(g: CsrGraph, source: int) -> BfsResult:
    """engine.py:440-475 on device: top-down level-synchronous traversal, then
    the queue BFS's parents (``_kernels.py:26-54``: the neighbour that discovers
    a vertex first in queue order) from the level array
    (``rb_bfs_first_parents``), so levels and predecessor equal the reference's."""
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")
    with BfsEngine(g, BfsParams(mode="sequential"), record_levels=True) as eng:
        res = eng.run(source)
        if len(res.levels) > 1:  # (an isolated source has no tree to order)
            torch = _lib.require_cuda()
            n_dev = eng.n_dev
            rs, col = g.device_arrays()[:2]
            par = torch.empty(n_dev, dtype=torch.int32, device="cuda")
            _lib.check(_lib.lib().rb_bfs_first_parents(_lib.ptr(rs), _lib.ptr(col), n_dev, _lib.ptr(eng.level_device()),
                                                       int(source), len(res.levels), _lib.ptr(par), _lib.stream_ptr()),
                       "rb_bfs_first_parents")
            res.predecessor[:n_dev] = par.cpu().numpy()
    for r in res.levels:
        r.wall_time = 0.0
    return res


# ---------------------------------------------------------------------------
# single steps (engine.py:252-429): explicit state in, mutated state out


def _step_engine(g: CsrGraph, reverse: bool) -> _DeviceBfs:
    cache = g._cache
    key = ("step_engine", reverse)
    if key not in cache:
        cache[key] = _DeviceBfs(g, hybrid=True, alpha=64, beta=8, g_bu=None, bu_reverse=reverse, trim_isolated=False)
    return cache[key]


def _run_step(g: CsrGraph, direction: int, frontier: Frontier, visited: Bitmap, parent: np.ndarray, reverse=True):
    torch = _lib.require_cuda()
    eng = _step_engine(g, reverse)
    n = g.n
    if n == 0:
        return Bitmap(0), np.zeros(3, np.int64)
    fr = frontier.to_bitmap_form()
    nw = (n + 31) // 32
    vis_in = torch.from_numpy(np.ascontiguousarray(visited.words32()).view(np.int32)).cuda()
    fr_in = torch.from_numpy(np.ascontiguousarray(fr.bits.words32()).view(np.int32)).cuda()
    par_in = torch.from_numpy(np.ascontiguousarray(parent, dtype=np.int32)).cuda()
    vis_out = torch.empty(nw, dtype=torch.int32, device="cuda")
    nxt_out = torch.empty(nw, dtype=torch.int32, device="cuda")
    par_out = torch.empty(n, dtype=torch.int32, device="cuda")
    ctr = np.zeros(3, np.int64)
    _lib.check(
        _lib.lib().rb_bfs_step(eng.h, direction, _lib.ptr(vis_in), _lib.ptr(fr_in), _lib.ptr(par_in),
                               _lib.ptr(vis_out), _lib.ptr(nxt_out), _lib.ptr(par_out),
                               ctr.ctypes.data_as(ctypes.c_void_p), _lib.stream_ptr()),
        "rb_bfs_step",
    )
    visited.w32[:nw] = vis_out.cpu().numpy().view(np.uint32)
    parent[:] = par_out.cpu().numpy()
    nxt = Bitmap.from_words32(n, nxt_out.cpu().numpy().view(np.uint32))
    return nxt, ctr


def top_down_step(g, frontier, visited, parent, threads: int = 1, pool=None):
    """engine.py:252-286: claim all unvisited neighbours of the frontier."""
    nxt, c = _run_step(g, 0, frontier, visited, parent)
    st = StepStats(n_next=int(c[0]), deg_next=int(c[1]), scanned_edges=int(c[2]),
                   per_thread_edges=_split_even(int(c[2]), threads))
    return Frontier.from_queue(g.n, nxt.to_indices()), st


def top_down_step_balanced(g, frontier, visited, parent, threads: int = 1, pool=None):
    """engine.py:289-323: the device scheduler already splits hubs across warps."""
    return top_down_step(g, frontier, visited, parent, threads, pool)


def bottom_up_step(g, frontier, visited, parent, threads: int = 1, pool=None):
    """engine.py:341-370: every unvisited vertex adopts a frontier neighbour."""
    nxt, c = _run_step(g, 1, frontier, visited, parent)
    st = StepStats(n_next=int(c[0]), deg_next=int(c[1]), scanned_edges=int(c[2]),
                   per_thread_edges=_split_even(int(c[2]), threads))
    return Frontier.from_bitmap(nxt), st


def bottom_up_step_balanced(g, frontier, visited, parent, ps=None, threads: int = 1, pool=None):
    """engine.py:373-398 (partition set accepted for API compatibility)."""
    return bottom_up_step(g, frontier, visited, parent, threads, pool)


def bottom_up_step_reduced(g_desc, frontier, visited, parent, ps=None, threads: int = 1, pool=None):
    """engine.py:401-429: scan the descending-degree rows forward (Alg. 6 order)."""
    nxt, c = _run_step(g_desc, 1, frontier, visited, parent, reverse=False)
    st = StepStats(n_next=int(c[0]), deg_next=int(c[1]), scanned_edges=int(c[2]),
                   per_thread_edges=_split_even(int(c[2]), threads))
    return Frontier.from_bitmap(nxt), st


def write_level_trace(results, path) -> None:
    """engine.py:620-639."""
    fields = ["round", "source", "mode", "level", "direction", "n_f", "m_f", "m_u", "scanned_edges",
              "wall_time_s", "pass1_hits", "live_vertices"]
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(fields)
        for rnd, res in enumerate(results):
            for rec in res.levels:
                w.writerow([
                    rnd, res.source, res.mode, rec.level, rec.direction, rec.n_f, rec.m_f, rec.m_u,
                    rec.scanned_edges, f"{rec.wall_time:.6f}",
                    "" if rec.pass1_hits is None else rec.pass1_hits,
                    "" if rec.live_vertices is None else rec.live_vertices,
                ])
