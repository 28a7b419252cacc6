"""CPU restatement of the z-slab exchange protocol (test infrastructure).

The device runtime (csrc/pn_runtime.cu: halo_exchange, gather_partials) does
these two steps with NCCL; the gloo tests (test_distributed.py) run this
restatement at world size 2 to pin the pairing, the stencil reach and the
rank-count-independent reduction order against the single-process oracle.
"""

import numpy as np


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
