"""ctypes binding of ``librcmbfs_b200.so`` (declared in include/rcmbfs_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, :func:`lib` / :func:`require_cuda` raise ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

RB_OK, RB_ERR_ARG, RB_ERR_CUDA, RB_ERR_NCCL, RB_ERR_OOM = 0, 1, 2, 3, 4
RB_PART_EXACT, RB_PART_COUNT_PASS1, RB_PART_SHRINK = 1, 2, 4

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
SZ = ctypes.c_size_t


class LevelRecordC(ctypes.Structure):
    _fields_ = [
        ("level", I64), ("direction", I64), ("n_f", I64), ("m_f", I64), ("m_u", I64),
        ("scanned_edges", I64), ("t_ns", I64), ("n_next", I64), ("t_queue_ns", I64), ("reserved", I64),
        ("pass1_hits", I64), ("live_vertices", I64), ("claimed", I64), ("reserved2", I64),
    ]


class BfsParamsC(ctypes.Structure):
    _fields_ = [
        ("alpha", I32), ("beta", I32), ("hybrid", I32), ("bu_reverse", I32),
        ("n_policy", I64), ("m_directed", I64), ("record_levels", I32), ("reserved0", I32),
    ]


class PartitionC(ctypes.Structure):
    _fields_ = [("v_lo", I64), ("n_glob", I64), ("d_td_row_starts", P), ("d_td_col", P)]


_SIGS = {
    "rb_last_error": ([], ctypes.c_char_p),
    "rb_version": ([], ctypes.c_int),
    "rb_kronecker_generate": ([ctypes.c_int, I64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, P, P], ctypes.c_int),
    "rb_csr_workspace_bytes": ([I64, I64], SZ),
    "rb_csr_build": ([P, I64, I64, P, SZ, ctypes.POINTER(I64), ctypes.POINTER(I64), P], ctypes.c_int),
    "rb_csr_emit": ([P, I64, I64, P, P, P, P], ctypes.c_int),
    "rb_rcm_workspace_bytes": ([I64, I64], SZ),
    "rb_rcm": ([P, P, P, I64, P, SZ, P, P, ctypes.POINTER(I64), P, ctypes.POINTER(I64), P], ctypes.c_int),
    "rb_permute_workspace_bytes": ([I64, I64], SZ),
    "rb_apply_permutation": ([P, P, P, I64, I64, P, P, P, SZ, P, P, P, P], ctypes.c_int),
    "rb_degree_sort_adjacency": ([P, P, P, I64, I64, ctypes.c_int, P, SZ, P, P], ctypes.c_int),
    "rb_bfs_create": ([P, P, P, P, I64, P, ctypes.POINTER(BfsParamsC), ctypes.POINTER(P)], ctypes.c_int),
    "rb_bfs_destroy": ([P], ctypes.c_int),
    "rb_bfs_create_part": ([P, P, P, P, I64, P, ctypes.POINTER(BfsParamsC), ctypes.POINTER(PartitionC),
                            ctypes.POINTER(P)], ctypes.c_int),
    "rb_bfs_reset_part": ([P, I64, P], ctypes.c_int),
    "rb_bfs_dist_level": ([P, I64, ctypes.c_int, ctypes.c_int, P, P, ctypes.POINTER(P), P, P], ctypes.c_int),
    "rb_bfs_words": ([P, ctypes.POINTER(I64), ctypes.POINTER(I64)], ctypes.c_int),
    "rb_make_nz": ([P, I64, P, P], ctypes.c_int),
    "rb_transpose_workspace_bytes": ([I64, I64], SZ),
    "rb_transpose_rows": ([P, P, I64, I64, I64, I64, P, SZ, P, P, P], ctypes.c_int),
    "rb_bfs_reset": ([P, I64, P], ctypes.c_int),
    "rb_bfs_set_partitions": ([P, P, I64, I64, I32], ctypes.c_int),
    "rb_bfs_xchg_alloc": ([P, I32, I32], ctypes.c_int),
    "rb_kronecker_generate_range": ([ctypes.c_int, I64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, I64, I64, P, P], ctypes.c_int),
    "rb_csr_keys": ([P, ctypes.POINTER(P), ctypes.POINTER(I64)], ctypes.c_int),
    "rb_keys_workspace_bytes": ([I64], SZ),
    "rb_keys_sort_unique": ([P, I64, ctypes.c_int, P, SZ, ctypes.POINTER(I64), P], ctypes.c_int),
    "rb_keys_to_csr": ([P, I64, I64, I64, P, P, P, P], ctypes.c_int),
    "rb_relabel_keys": ([P, P, I64, I64, P, P, P], ctypes.c_int),
    "rb_bfs_xchg_handle_bytes": ([], SZ),
    "rb_bfs_xchg_handle": ([P, P], ctypes.c_int),
    "rb_bfs_xchg_open": ([P, P], ctypes.c_int),
    "rb_bfs_xchg_connect_local": ([P, I32], ctypes.c_int),
    "rb_bfs_dist_reset": ([P, I64, I64, P], ctypes.c_int),
    "rb_bfs_dist_traverse": ([P, P], ctypes.c_int),
    "rb_bfs_dist_traverse_emu": ([P, I32, P], ctypes.c_int),
    "rb_bfs_dist_results": ([P, P, I64, ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_double), P], ctypes.c_int),
    "rb_bfs_traverse": ([P, P], ctypes.c_int),
    "rb_bfs_elapsed": ([P, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "rb_bfs_results": ([P, P, P, P, I64, ctypes.POINTER(I64), P], ctypes.c_int),
    "rb_bfs_results_async": ([P, P, P, I64, P, I32, P], ctypes.c_int),
    "rb_bfs_wait": ([P, I32], ctypes.c_int),
    "rb_bfs_complete": ([P, P, P, I64, ctypes.POINTER(I64)], ctypes.c_int),
    "rb_bfs_state_bytes": ([], SZ),
    "rb_bfs_step": ([P, ctypes.c_int, P, P, P, P, P, P, P, P], ctypes.c_int),
    "rb_bfs_parent_ptr": ([P], P),
    "rb_bfs_level_ptr": ([P], P),
    "rb_bfs_grid": ([P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "rb_bfs_barrier_probe": ([P, ctypes.c_int, ctypes.POINTER(ctypes.c_double), P], ctypes.c_int),
    "rb_bfs_debug_timestamps": ([P, P, I64, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "rb_components": ([P, P, I64, P, I64, P, P], ctypes.c_int),
    "rb_chunglu_workspace_bytes": ([I64], SZ),
    "rb_chunglu_generate": ([P, I64, I64, ctypes.c_uint64, P, SZ, P, P], ctypes.c_int),
    "rb_validate_workspace_bytes": ([I64], SZ),
    "rb_validate": ([P, P, I64, P, I64, P, P, SZ, P, P, P], ctypes.c_int),
    "rb_bfs_first_parents": ([P, P, I64, P, I64, I64, P, P], ctypes.c_int),
    "rb_host_fill_i32": ([P, I64, ctypes.c_int32, ctypes.c_int], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)


def load(path: str | None = None, build: bool = True):
    """Load (building first if stale) and bind the C-ABI library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if path is None and os.environ.get("RB_LIB"):
            path = os.environ["RB_LIB"]  # tuning variants built with _build --out
            build = False
        if path is None:
            path = _build.LIB
            if build and os.environ.get("RB_NO_BUILD") != "1":
                _build.build()
        if not os.path.exists(path):
            raise RuntimeError(f"CUDA extension {path} is missing; run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def lib():
    return load()


class CudaError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == RB_OK:
        return
    msg = (lib().rb_last_error() or b"").decode(errors="replace")
    if rc == RB_ERR_ARG:
        raise ValueError(msg or what)
    if rc == RB_ERR_OOM:
        raise MemoryError(f"{what}: {msg}")
    raise CudaError(f"{what}: {msg} (code {rc})")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2012_10026_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    lib()
    return torch


def workspace(nbytes: int, device="cuda"):
    """A uint8 CUDA scratch tensor.  Large requests first hand torch's cached
    but unused blocks back to the driver: at scale 27 the relabel's 96 GB
    workspace fits the GPU, but not next to 60 GB of cached fragments."""
    import torch

    if nbytes >= (8 << 30):
        torch.cuda.empty_cache()
    try:
        return torch.empty(nbytes, dtype=torch.uint8, device=device)
    except torch.OutOfMemoryError:
        torch.cuda.empty_cache()
        return torch.empty(nbytes, dtype=torch.uint8, device=device)


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())
