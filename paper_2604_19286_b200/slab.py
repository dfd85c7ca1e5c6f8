"""Slab decomposition of the grid along axis 0 and the ghost-plane reduction.

DESIGN.md §Multi-GPU.  Rank r owns cells and nodes with ix in
[x_begin, x_end) and only the particles located in those cells (particles
owned by cell).  mm_assemble writes node rows outside the slab into ghost
planes (order 1: plane x_end; order 2: x_begin-1, x_end, x_end+1), which are
the only data exchanged: they are sent to the slab neighbours (periodic ring)
over torch.distributed (NCCL on GPUs, gloo in the CPU tests) and added into
the owner's rows by the mm_ghost_add kernel.

The bookkeeping here is pure index arithmetic on planes; the `add` callback
defaults to the CUDA kernel (mm_ghost_add).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def slab_bounds(n0: int, world: int, rank: int):
    """Balanced contiguous split of n0 cell planes over `world` ranks."""
    base, extra = divmod(n0, world)
    xb = rank * base + min(rank, extra)
    return xb, xb + base + (1 if rank < extra else 0)


def ghost_routes(order: int, width: int):
    """(ghost plane index, direction, owner plane index) triples.

    direction -1: the owner is rank r-1 and the plane is its LAST-k plane
    (owner index relative to the owner's x_begin is computed by the receiver:
    width_prev - 1); direction +1: the owner is rank r+1, planes 0.. of it."""
    if order == 1:
        return [(0, +1, 0)]
    return [(0, -1, -1), (1, +1, 0), (2, +1, 1)]


def exchange_ghosts(out: torch.Tensor, ghost: torch.Tensor, order: int, plane_elems: int, rank: int,
                    world: int, widths, add=None, group=None):
    """Sum ghost planes into their owners.

    out    [width * plane_elems] owned rows of this rank (any shape, contiguous)
    ghost  [nghost * plane_elems] ghost planes of this rank
    widths slab width of every rank (for the -1 direction's target plane)
    add    add(k, src): add one received plane `src` into owned plane k (relative to x_begin).
           The product path passes the mm_ghost_add kernel; the CPU tests a torch add.
    """
    g = ghost.reshape(-1, plane_elems)
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    send_next = [k for k, d, _ in ghost_routes(order, widths[rank]) if d == +1]
    send_prev = [k for k, d, _ in ghost_routes(order, widths[rank]) if d == -1]
    recv_from_prev = torch.empty((len(send_next), plane_elems), dtype=ghost.dtype, device=ghost.device)
    recv_from_next = torch.empty((len(send_prev), plane_elems), dtype=ghost.dtype, device=ghost.device)
    ops = []
    if send_next:
        ops.append(dist.P2POp(dist.isend, g[send_next[0]:send_next[-1] + 1].contiguous(), nxt, group))
        ops.append(dist.P2POp(dist.irecv, recv_from_prev, prv, group))
    if send_prev:
        ops.append(dist.P2POp(dist.isend, g[send_prev[0]:send_prev[-1] + 1].contiguous(), prv, group))
        ops.append(dist.P2POp(dist.irecv, recv_from_next, nxt, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    # planes from r-1 (its x_end, x_end+1) are my planes 0, 1; planes from r+1 (its x_begin-1) my last plane
    for k in range(len(send_next)):
        add(k, recv_from_prev[k])
    for k in range(len(send_prev)):
        add(widths[rank] - 1 - k, recv_from_next[k])
    return out
