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
        obs_dev.device.index or 0, ctypes.c_void_p(st.cuda_stream or 0x1)))  # 0x1: legacy
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


class GatherPlan:
    """Where every row of the gathered per-rank payloads goes in the global order.

    Built once per (order, world size); the gather itself is then one collective plus
    one device scatter (no host index work inside a timed step).
    sizes[r] = receivers of rank r, cap = max(sizes); dest (world*cap,) holds the global
    receiver index of each gathered row, n_total for padding rows.
    """

    def __init__(self, order, world_size: int, n_total: int, tile: int | None = None):
        import torch
        tile = tile_size() if tile is None else tile
        self.world_size, self.n_total = world_size, n_total
        self.sizes = [rank_tiles(n_total, r, world_size, tile).size for r in range(world_size)]
        self.cap = max(self.sizes) if self.sizes else 0
        dev = order.device if hasattr(order, "device") else "cpu"
        dest = torch.full((world_size * self.cap,), n_total, dtype=torch.long, device=dev)
        for r in range(world_size):
            idx = rank_indices(order, r, world_size, tile)
            idx = torch.as_tensor(idx, device=dev).long()
            dest[r * self.cap:r * self.cap + self.sizes[r]] = idx
        self.dest = dest


def gather_field(acc, evals, order, rank: int, world_size: int, n_total: int, group=None,
                 tile: int | None = None, plan: GatherPlan | None = None):
    """Gather per-rank (acc, evals) to rank 0 and scatter them into global order.

    acc is (n_local, F) complex128, evals (n_local,) int64, both in the rank's
    tile order.  Returns (acc_full, evals_full) on rank 0, (None, None) elsewhere.
    Works for NCCL (CUDA tensors, one dist.gather to rank 0) and gloo (CPU tensors).
    `plan` (GatherPlan of the same order/world) is built on the fly if not given.
    """
    import torch
    import torch.distributed as dist
    if plan is None:
        plan = GatherPlan(order, world_size, n_total, tile)
    F = acc.shape[1]
    cap = plan.cap
    # complex -> float64 (NCCL has no complex type); evals ride as float64 bits
    pay = torch.zeros((cap, 2 * F + 1), dtype=torch.float64, device=acc.device)
    n_loc = acc.shape[0]
    pay[:n_loc, :2 * F] = torch.view_as_real(acc).reshape(n_loc, 2 * F)
    pay[:n_loc, 2 * F] = evals.view(torch.float64)
    # one gather to rank 0 (only rank 0 receives the field: W x fewer bytes than an
    # all-gather); gloo gathers host tensors
    host = dist.get_backend(group) == "gloo"
    src = pay.cpu() if host else pay
    bufs = [torch.empty_like(src) for _ in range(world_size)] if rank == 0 else None
    dist.gather(src, gather_list=bufs, dst=0, group=group)
    if rank != 0:
        return None, None
    allp = torch.cat(bufs).to(acc.device)
    dest = plan.dest.to(acc.device)
    out = torch.zeros((n_total + 1, 2 * F + 1), dtype=torch.float64, device=acc.device)
    out[dest] = allp  # padding rows land in the extra row n_total
    acc_full = torch.view_as_complex(out[:n_total, :2 * F].reshape(n_total, F, 2).contiguous())
    evals_full = out[:n_total, 2 * F].contiguous().view(torch.int64)
    return acc_full, evals_full
