"""z-slab decomposition of the P_N solve across the GPUs of one node.

One process per GPU (torchrun), one device context per rank owning the
global planes [z0, z0 + nz_local).  The device runtime (pn_runtime.cu) does
the exchange itself: before every stencil apply the first / last plane of the
input vector goes to the lower / upper neighbour's halo plane (NCCL
send/recv), and every reduction folds its block partials into per-plane sums
that are all-gathered, so all ranks sum the same nz numbers in the same order.

This module holds the host side: slab bounds, NCCL-id distribution through
torch.distributed, the per-rank context, and CPU reference implementations of
the two exchange steps (used by the gloo tests to pin the protocol; the device
path never calls them).
"""

from __future__ import annotations

import numpy as np

from .program import as_tables


def slab_bounds(nz, world, rank):
    """(z0, nz_local) of `rank`: equal slabs (nz % world == 0, as NCCL
    all-gather of plane sums needs equal counts)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world")
    if nz % world:
        raise ValueError(f"nz={nz} must be divisible by the number of GPUs ({world})")
    n = nz // world
    return rank * n, n


def share_nccl_id(rank, world):
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    import torch.distributed as dist
    from . import _lib
    buf = [None]
    if rank == 0:
        raw = np.zeros(128, np.uint8)
        _lib.check(_lib.load().pn_nccl_unique_id(raw.ctypes.data))
        buf[0] = bytes(raw)
    if world > 1:
        dist.broadcast_object_list(buf, src=0)
    return buf[0]


def make_rank_context(program_or_N, spec, rank, world, device=None, nccl_id=None):
    """Create and fill this rank's slab context (the fields are the global
    arrays; the context uploads and transposes its slab)."""
    from .solver import PnContext
    tables = as_tables(program_or_N)
    z0, nzl = slab_bounds(spec.res[2], world, rank)
    if world > 1 and nccl_id is None:
        nccl_id = share_nccl_id(rank, world)
    ctx = PnContext(tables, spec.res, spec.h, device=rank if device is None else device, z0=z0, nz_local=nzl,
                    rank=rank, world=world, nccl_id=nccl_id if world > 1 else None)
    ctx.set_fields(spec)
    return ctx


def gather_slabs(local, rank, world):
    """All slabs of a vector on every rank (z is the slowest index, so the
    global vector is the concatenation in rank order)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts)


# ---------------------------------------------------------------------------
# CPU reference of the exchange protocol (tests only)
# ---------------------------------------------------------------------------

def exchange_halos_cpu(local, plane, rank, world):
    """Halo planes of a local slab vector (1-D torch tensor, z slowest):
    returns (lower, upper), zeros at the global boundary.  Same pairing as
    the device code: send first plane down / receive lower halo, send last
    plane up / receive upper halo."""
    import torch
    import torch.distributed as dist
    lower = torch.zeros(plane, dtype=local.dtype)
    upper = torch.zeros(plane, dtype=local.dtype)
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, local[:plane].contiguous(), rank - 1))
        ops.append(dist.P2POp(dist.irecv, lower, rank - 1))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, local[-plane:].contiguous(), rank + 1))
        ops.append(dist.P2POp(dist.irecv, upper, rank + 1))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return lower, upper


def plane_sum_reduce_cpu(values, plane, z0, nz, world):
    """Deterministic reduction of sum(values) where `values` is this rank's
    slab of a per-unknown quantity: per-plane sums (fixed order), all-gather,
    sum in plane order.  Independent of the rank count bit for bit."""
    import torch
    import torch.distributed as dist
    nzl = values.numel() // plane
    local = torch.tensor([float(np.sum(values[k * plane:(k + 1) * plane].numpy())) for k in range(nzl)],
                         dtype=torch.float64)
    if world > 1:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local)
        allp = torch.cat(parts)
    else:
        allp = local
    acc = 0.0
    for v in allp.tolist():
        acc = acc + v
    return acc
