"""Slab decomposition of the grid along axis 0 and the ghost-plane reduction.

DESIGN.md §Multi-GPU.  Rank r owns cells and nodes with ix in
[x_begin, x_end) and only the particles located in those cells (particles
owned by cell).  mm_assemble writes node rows outside the slab into ghost
planes (order 1: plane x_end; order 2: x_begin-1, x_end, x_end+1), which are
the only data exchanged: they are sent to the slab neighbours (periodic ring)
over torch.distributed (NCCL on GPUs, gloo in the CPU tests) and added into
the owner's rows by the mm_ghost_add kernel.

The product path does the ghost reduction inside libmm (mm_assemble_slab /
mm_ghost_exchange over an mm_comm, NCCL send/recv on the library's comm stream,
overlapped with the interior bins).  exchange_ghosts below is the same routing
table over torch.distributed: the CPU (gloo) tests check the multi-rank routing
with it, which one GPU cannot do with NCCL.
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
    add    add(k, src): add one received plane `src` into owned plane k (relative to x_begin),
           e.g. the mm_ghost_add kernel or a torch add (required).
    """
    if add is None:
        raise ValueError("exchange_ghosts needs an add(k, src) callback")
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


def migrate(pos: torch.Tensor, q: torch.Tensor, B, rank: int, world: int, partition, group=None,
            max_rounds: int | None = None):
    """Send the particles that left this rank's slab towards their owners and return this rank's
    new (pos, q, B): the particles that stayed, then those received, in a deterministic order.

    The "sort & communicate" stage of the PIC cycle: after
    the mover, particles are owned by cell again before mm_sort_by_cell.
    partition(pos, q, B) -> (pos_o, q_o, B_o, (n_stay, n_prev, n_next)): the stable 3-way
    partition (mm_slab_partition on GPUs; a torch stand-in in the CPU tests) sends a particle
    outside the slab towards the nearer side of the periodic ring.

    Multi-hop: a particle that moved further than the neighbouring slab is forwarded again in
    the next round; rounds repeat until the all-reduced number of leavers is 0 (at most about
    world / 2 + 1 rounds, each one hop).  Per round: the two leaver counts, then the packed
    leavers [n, 7] (or [n, 4] without B) to each neighbour, posted next-first."""
    if world == 1:
        pos_o, q_o, B_o, _ = partition(pos, q, B)
        return pos_o, q_o, B_o
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    dev = pos.device
    keep_p, keep_q, keep_B = [], [], []
    cur = (pos, q, B)
    limit = max_rounds if max_rounds is not None else world + 1
    for _ in range(limit + 1):
        pos_o, q_o, B_o, (ns, npv, nnx) = partition(*cur)
        keep_p.append(pos_o[:ns])
        keep_q.append(q_o[:ns])
        if B_o is not None:
            keep_B.append(B_o[:ns])
        total = torch.tensor([npv + nnx], dtype=torch.int64, device=dev)
        dist.all_reduce(total, group=group)
        if int(total.item()) == 0:
            break

        def pack(a, b):
            cols = [pos_o[a:b], q_o[a:b, None]] + ([B_o[a:b]] if B_o is not None else [])
            return torch.cat(cols, dim=1).contiguous()

        to_prev, to_next = pack(ns, ns + npv), pack(ns + npv, ns + npv + nnx)
        c_next = torch.tensor([nnx], dtype=torch.int64, device=dev)
        c_prev = torch.tensor([npv], dtype=torch.int64, device=dev)
        r_prev = torch.zeros(1, dtype=torch.int64, device=dev)   # count coming from r-1 (its to_next)
        r_next = torch.zeros(1, dtype=torch.int64, device=dev)   # count coming from r+1 (its to_prev)
        ops = [dist.P2POp(dist.isend, c_next, nxt, group), dist.P2POp(dist.irecv, r_prev, prv, group),
               dist.P2POp(dist.isend, c_prev, prv, group), dist.P2POp(dist.irecv, r_next, nxt, group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        ncol = to_next.shape[1]
        from_prev = torch.empty((int(r_prev.item()), ncol), dtype=pos.dtype, device=dev)
        from_next = torch.empty((int(r_next.item()), ncol), dtype=pos.dtype, device=dev)
        ops = []
        if nnx:
            ops.append(dist.P2POp(dist.isend, to_next, nxt, group))
        if from_prev.shape[0]:
            ops.append(dist.P2POp(dist.irecv, from_prev, prv, group))
        if npv:
            ops.append(dist.P2POp(dist.isend, to_prev, prv, group))
        if from_next.shape[0]:
            ops.append(dist.P2POp(dist.irecv, from_next, nxt, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        got = torch.cat([from_prev, from_next], dim=0)
        cur = (got[:, 0:3].contiguous(), got[:, 3].contiguous(),
               got[:, 4:7].contiguous() if B_o is not None else None)
    else:
        raise RuntimeError(f"migration did not converge in {limit} rounds")
    new_pos = torch.cat(keep_p, dim=0).contiguous()
    new_q = torch.cat(keep_q, dim=0).contiguous()
    new_B = torch.cat(keep_B, dim=0).contiguous() if B is not None else None
    return new_pos, new_q, new_B
