"""Receiver-tile partition of the GBS stage across GPUs (one process per GPU).

SURVEY.md 8(e): each receiver's sum depends on all beams and on nothing else
(kernels.py:364-399), so receivers shard with no data-path exchange -- the
reference's observer-range split across workers (parallel.py:108-140), re-cut
as SPATIAL tiles: the global Hilbert order (bf_tile_order_dev) is cut into
tiles of bf_tile_size() receivers, dealt round-robin to the ranks (balancing
the spatially varying tie-path / cutoff density), and every rank sums its
tiles with the presorted flag so the kernel's tiles ARE the global tiles.
A receiver's result is therefore bit-identical for any number of ranks.

The only collective is the final gather of the per-rank field tiles to rank 0
(torch.distributed over NCCL/NVLink; gloo on CPU for the tests).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def world(group=None):
    """(world_size, rank) of the default / given process group, (1, 0) if none."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def tile_size() -> int:
    return int(_lib.load().bf_tile_size())


def tile_order(obs_dev):
    """Global spatial order of device observers (int64 CUDA tensor of indices)."""
    import torch
    n = obs_dev.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=obs_dev.device)
    st = torch.cuda.current_stream(obs_dev.device)
    _lib.check(_lib.load().bf_tile_order_dev(
        ctypes.c_void_p(obs_dev.data_ptr()), n, ctypes.c_void_p(perm.data_ptr()),
        obs_dev.device.index or 0, ctypes.c_void_p(st.cuda_stream)))
    return perm.long()


def rank_tiles(n: int, rank: int, world_size: int, tile: int | None = None) -> np.ndarray:
    """Positions (into the global tile order) owned by `rank`: tiles rank, rank+W, ..."""
    tile = tile_size() if tile is None else tile
    n_tiles = -(-n // tile)
    mine = np.arange(rank, n_tiles, world_size)
    if mine.size == 0:
        return np.zeros(0, np.int64)
    pos = (mine[:, None] * tile + np.arange(tile)[None, :]).reshape(-1)
    return pos[pos < n]


def rank_indices(order, rank: int, world_size: int, tile: int | None = None):
    """Observer indices owned by `rank`, in tile order (same device/type as `order`)."""
    pos = rank_tiles(int(order.shape[0]), rank, world_size, tile)
    if hasattr(order, "index_select"):
        import torch
        return order.index_select(0, torch.from_numpy(pos).to(order.device))
    return np.asarray(order)[pos]


def gather_field(acc, evals, order, rank: int, world_size: int, n_total: int, group=None,
                 tile: int | None = None):
    """Gather per-rank (acc, evals) to rank 0 and scatter them into global order.

    acc is (n_local, F) complex128, evals (n_local,) int64, both in the rank's
    tile order.  Returns (acc_full, evals_full) on rank 0, (None, None) elsewhere.
    Works for NCCL (CUDA tensors) and gloo (CPU tensors).
    """
    import torch
    import torch.distributed as dist
    F = acc.shape[1]
    sizes = [rank_tiles(n_total, r, world_size, tile).size for r in range(world_size)]
    cap = max(sizes)
    # complex -> float64 (NCCL has no complex type); evals ride as float64 bits
    pay = torch.zeros((cap, 2 * F + 1), dtype=torch.float64, device=acc.device)
    n_loc = acc.shape[0]
    pay[:n_loc, :2 * F] = torch.view_as_real(acc).reshape(n_loc, 2 * F)
    pay[:n_loc, 2 * F] = evals.view(torch.float64)
    if pay.is_cuda and dist.get_backend(group) == "gloo":  # gloo gathers host tensors
        pay = pay.cpu()
    bufs = [torch.empty_like(pay) for _ in range(world_size)]
    dist.all_gather(bufs, pay, group=group)
    bufs = [b.to(acc.device) for b in bufs]
    if rank != 0:
        return None, None
    acc_full = torch.zeros((n_total, F), dtype=torch.complex128, device=acc.device)
    evals_full = torch.zeros(n_total, dtype=torch.int64, device=acc.device)
    for r in range(world_size):
        idx = rank_indices(order, r, world_size, tile)
        idx = torch.as_tensor(idx, device=acc.device).long()
        k = sizes[r]
        acc_full[idx] = torch.view_as_complex(bufs[r][:k, :2 * F].reshape(k, F, 2).contiguous())
        evals_full[idx] = bufs[r][:k, 2 * F].contiguous().view(torch.int64)
    return acc_full, evals_full
