"""World-size-2 gloo tests of the z-slab protocol (CPU): halo pairing,
stencil reach, global Dirichlet masks and rank-count-independent reductions,
checked against the single-process operator from the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_00410_b200.distributed import slab_bounds
from slab_protocol import exchange_halos_cpu, plane_sum_reduce_cpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, res, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
        from cases import probe_vector, rand_spec
        from oracle.oracle import StencilOracle
        from paper_1807_00410_b200.program import build_tables
        spec = rand_spec(N, res, seed)
        o = StencilOracle(build_tables(N), spec)
        A = o.csr()
        At = A.T.tocsr()
        nx, ny, nz = res
        U = (N + 1) ** 2
        plane = nx * ny * U
        z0, nzl = slab_bounds(nz, world, rank)
        x = probe_vector(o.R)
        local = torch.tensor(x[z0 * plane:(z0 + nzl) * plane])
        lower, upper = exchange_halos_cpu(local, plane, rank, world)
        # the slab's rows only reach one plane beyond the slab: apply them to
        # [lower halo | local | upper halo] and compare with the global product
        lo = max(z0 - 1, 0)
        hi = min(z0 + nzl + 1, nz)
        ext = np.concatenate(([lower.numpy()] if z0 > 0 else []) + [local.numpy()] +
                             ([upper.numpy()] if z0 + nzl < nz else []))
        rows = slice(z0 * plane, (z0 + nzl) * plane)
        ok = True
        for M in (A, At):
            sub = M[rows][:, lo * plane:hi * plane]
            full = M[rows]
            ok &= (full.nnz == sub.nnz)
            y_local = sub @ ext
            ok &= y_local.tobytes() == (M @ x)[rows].tobytes()
        # rank-count independent reductions
        w = A @ x
        s_dist = plane_sum_reduce_cpu(torch.tensor(w[rows] * w[rows]), plane, z0, nz, world)
        out[rank] = (bool(ok), s_dist)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,res", [(1, (5, 4, 6)), (3, (4, 3, 4)), (7, (3, 3, 4))])
def test_slab_protocol_world2_gloo(N, res):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, N, res, 5, out), nprocs=world, join=True)
    assert out[0][0] and out[1][0]
    # both ranks agree bit for bit, and equal the single-rank reduction
    assert out[0][1] == out[1][1]
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from cases import probe_vector, rand_spec
    from oracle.oracle import StencilOracle
    from paper_1807_00410_b200.program import build_tables
    o = StencilOracle(build_tables(N), rand_spec(N, res, 5))
    x = probe_vector(o.R)
    w = o.apply(x)
    plane = res[0] * res[1] * (N + 1) ** 2
    sums = [float(np.sum((w * w)[k * plane:(k + 1) * plane])) for k in range(res[2])]
    acc = 0.0
    for v in sums:
        acc = acc + v
    assert out[0][1] == acc


def test_slab_bounds():
    assert slab_bounds(256, 8, 3) == (96, 32)
    with pytest.raises(ValueError):
        slab_bounds(10, 4, 0)


def _digest_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        nz, plane = 12, 40
        z0, nzl = slab_bounds(nz, world, rank)
        x = np.random.default_rng(3).normal(size=nz * plane)
        parts = [None] * world
        dist.all_gather_object(parts, bench.plane_digests(x[z0 * plane:(z0 + nzl) * plane], nzl))
        out[rank] = bench.global_digest(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_solve_checksum_is_rank_count_independent(world):
    """bench.py's solve_check: per-plane digests gathered in rank order give
    the digest of the whole vector for any slab decomposition."""
    import bench
    nz, plane = 12, 40
    x = np.random.default_rng(3).normal(size=nz * plane)
    want = bench.global_digest([bench.plane_digests(x, nz)])
    out = mp.Manager().dict()
    mp.spawn(_digest_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert set(out.values()) == {want}


@pytest.mark.parametrize("nz,world", [(256, 2), (256, 8), (512, 8), (512, 4)])
def test_slab_planes_cover_each_rank(nz, world):
    """bench.slab_planes: each rank generates its slab plus the +1 plane its
    field upload reads (clamped at nz), and make_rank_context accepts it."""
    import bench
    for rank in range(world):
        z0, nzl, (k0, k1) = bench.slab_planes(nz, world, rank)
        assert (z0, nzl) == slab_bounds(nz, world, rank)
        assert k0 == z0 and k1 == min(z0 + nzl + 1, nz)


def test_rank_context_rejects_uncovered_planes():
    from paper_1807_00410_b200.configs import make_config
    from paper_1807_00410_b200.distributed import make_rank_context
    from paper_1807_00410_b200.program import build_tables
    spec = make_config(3, n=16, planes=(0, 8)).spec     # rank 1 of 2 needs planes 8..15
    with pytest.raises(ValueError, match="do not cover"):
        make_rank_context(build_tables(5), spec, rank=1, world=2)
