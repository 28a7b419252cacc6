"""z-slab decomposition of the P_N solve across the GPUs of one node.

One process per GPU (torchrun), one device context per rank owning the
global planes [z0, z0 + nz_local).  The device runtime (pn_runtime.cu) does
the exchange itself: before every stencil apply the first / last plane of the
input vector goes to the lower / upper neighbour's halo plane (NCCL
send/recv), and every reduction folds its block partials into per-plane sums
that are all-gathered, so all ranks sum the same nz numbers in the same order.

This module holds the host side: slab bounds, NCCL-id distribution through
torch.distributed and the per-rank context (solver.solve_pn(..., world,
rank) and bench.py build on it).  tests/slab_protocol.py restates the two
exchange steps on the CPU for the gloo tests.
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


def nccl_selftest(device=0, n=4096):
    """One-rank run of the NCCL call patterns of the slab path on this box
    (communicator, grouped send/recv, in-place all-gather, graph capture on a
    forked stream); raises on any failure.  pn_nccl_selftest in the C ABI."""
    from . import _lib
    _lib.check(_lib.load().pn_nccl_selftest(int(device), int(n)))


def make_rank_context(program_or_N, spec, rank, world, device=None, nccl_id=None):
    """Create and fill this rank's slab context.  The fields are the global
    arrays or this rank's planes (spec.z_planes, covering the slab and its
    +1 plane); the context uploads and transposes its slab."""
    from .solver import PnContext
    tables = as_tables(program_or_N)
    z0, nzl = slab_bounds(spec.res[2], world, rank)
    zp = getattr(spec, "z_planes", None)
    if zp is not None and not (zp[0] <= z0 and zp[0] + zp[1] >= min(z0 + nzl + 1, spec.res[2])):
        raise ValueError(f"spec planes {zp} do not cover slab [{z0}, {z0 + nzl}] of rank {rank}")
    if world > 1 and nccl_id is None:
        nccl_id = share_nccl_id(rank, world)
    ctx = PnContext(tables, spec.res, spec.h, device=rank if device is None else device, z0=z0, nz_local=nzl,
                    rank=rank, world=world, nccl_id=nccl_id if world > 1 else None)
    ctx.set_fields(spec)
    return ctx
