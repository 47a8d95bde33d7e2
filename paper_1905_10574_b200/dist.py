"""Multi-GPU solve: one process per GPU, tile columns block-cyclic (column j on rank j % R).

Host side of the exchange described in DESIGN.md §7 (the reference has no distributed mode,
SPEC.md:308; BASELINE north_star: "tile columns of Y are distributed block-cyclically; solved
tiles and their scale factors are pushed to dependent GPUs over NVLink"):

1. ``rsylv_b200_dist_prepare``: every rank packs A, B (replicated) and its workspace, validates,
   and exports CUDA-IPC handles of the buffers its peers write into.
2. all-gather of the handles, status agreement, barrier (nobody pushes into a peer that has not
   reset its flags yet).
3. ``rsylv_b200_dist_run``: the persistent kernel on the owned columns; each solved tile is
   pushed (st.global over NVLink + st.release.sys flag) to every rank owning a column to its
   right, where it is a row-update source. Returns the local exponent minimum and norm.
4. NCCL all-reduce MIN of the exponent minima and MAX of the (re-based) tile norms -> the global
   alpha (tile_grid.cpp:38-42 across GPUs).
5. ``rsylv_b200_dist_finish``: consistency scaling + copy-out of the owned columns.

The pure-Python pieces (ownership, push targets, alpha reduction) are unit-tested on CPU with a
2-rank gloo group (tests/test_dist_host.py); the device exchange itself is validated on one GPU
with virtual ranks (tests/test_gpu_multirank.py).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as nat


def owner(j: int, nranks: int) -> int:
    """Rank that owns tile column j."""
    return j % nranks


def push_targets(j: int, ncols: int, nranks: int, rank: int) -> list[int]:
    """Ranks that receive solved tile (i, j) of `rank` (mirror of push_tile in kernels.cu):
    every other rank owning a column j' > j."""
    out = []
    for r in range(nranks):
        if r == rank:
            continue
        first = j + 1 + ((r - (j + 1) % nranks) + nranks) % nranks
        if first < ncols:
            out.append(r)
    return out


def alpha_exponent(emin: int, numax: float, omega: float) -> int:
    """Largest alpha = 2^(emin + s), s >= 0, with numax * 2^s <= omega and alpha <= 1
    (mirror of alpha_exponent in runtime.cpp)."""
    s = -emin
    if numax > 0.0:
        mn, en = math.frexp(numax)
        mo, eo = math.frexp(omega)
        smax = eo - en - (0 if mn <= mo else 1)
        s = max(0, min(s, smax))
    return emin + s


def reduce_alpha(emin_local: int, numax_local: float, omega: float, dist, device=None):
    """All-reduce MIN of the exponent minima, then MAX of the norms re-based to the global
    minimum; returns (alpha_exp, emin_global, numax_global)."""
    import torch
    dev = device if device is not None else "cpu"
    t = torch.tensor([emin_local], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    emin_g = int(t.item())
    rebased = math.ldexp(numax_local, emin_g - emin_local) if numax_local > 0 else 0.0
    t = torch.tensor([rebased], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    numax_g = float(t.item())
    return alpha_exponent(emin_g, numax_g, omega), emin_g, numax_g


def solve_dist(A, a_codes, B, b_codes, Cm, Y, tile_size: int, cfg=None, stream=None,
               device: int = 0):
    """Distributed solve over the default torch.distributed group (NCCL). A, B, C are the full
    (replicated) column-major CUDA tensors of this rank; on return Y holds this rank's columns.
    Returns (status, alpha_exp, nat.Result)."""
    import torch
    import torch.distributed as dist
    from .api import OverflowConfig
    cfg = cfg or OverflowConfig()
    R, r = dist.get_world_size(), dist.get_rank()
    L, ctx = nat.lib(), nat.context(device)
    m, n = Cm.shape
    opt = nat.Options(cfg.omega, cfg.small_num, int(tile_size), 0, 1)
    res = nat.Result()
    handle = (C.c_ubyte * nat.DIST_HANDLE_BYTES)()
    up = lambda x: np.ascontiguousarray(x, dtype=np.uint8).ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
    st = L.rsylv_b200_dist_prepare(ctx, R, r, m, n, C.c_void_p(A.data_ptr()), A.stride(1),
                                   up(a_codes), C.c_void_p(B.data_ptr()), B.stride(1),
                                   up(b_codes), C.c_void_p(Cm.data_ptr()), Cm.stride(1),
                                   C.byref(opt), C.c_void_p(stream) if stream else None,
                                   handle, C.byref(res))
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([st], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if int(t.item()) != nat.RSYLV_OK:
        return int(t.item()), 0, res
    handles = [None] * R
    dist.all_gather_object(handles, bytes(handle))
    blob = b"".join(handles)
    torch.cuda.synchronize()
    dist.barrier()
    blob_buf = C.create_string_buffer(blob, len(blob))
    st = L.rsylv_b200_dist_run(ctx, C.cast(blob_buf, C.c_void_p),
                               C.c_void_p(stream) if stream else None, C.byref(res))
    t = torch.tensor([st], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if int(t.item()) != nat.RSYLV_OK:
        return int(t.item()), 0, res
    ae, emin_g, numax_g = reduce_alpha(int(res.alpha_exp), float(res.max_tile_norm),
                                       cfg.omega, dist, device=dev)
    res.alpha_exp = emin_g
    res.max_tile_norm = numax_g
    st = L.rsylv_b200_dist_finish(ctx, ae, C.c_void_p(Y.data_ptr()), Y.stride(1),
                                  C.c_void_p(stream) if stream else None, C.byref(res))
    return st, ae, res
