"""Drop-in B200 runtime for the reference's solve path.

Mirrors pnrte's runtime entry points (pkg/src/pnrte/__init__.py:21-25):

    assemble(program, spec)                                   solver.py:96
    solve_normal_cg(system, tol=1e-8, max_iter=50000,
                    primal_tol=None, jacobi=False, x0=None)   solver.py:189-190
    unstagger(u, program, res)                                solver.py:275
    SparseSystem, SolveReport                                 solver.py:34-50

with the same argument meaning, result types and error behaviour (ValueError
for tol <= 0 or a dim mismatch, non-convergence reported in the report, zero
RHS returns x = 0 converged).  ``assemble`` does not build a CSR matrix: it
creates a device context holding the stencil tables and the fields, and the
system's ``A`` is a matrix-free operator (``A @ x``, ``A.T @ x`` run the sm_100a
kernels; ``A.to_scipy()`` exports the exact CSR, assembled on the device, for
parity checks).  Neumann specs get an explicit device CSR (CsrOperator).

Extra keyword arguments (all optional): ``mode`` ("fast" | "faithful"),
``device`` and, for faithful runs, ``blas_threads`` / ``blas_kernel`` (the
OpenBLAS configuration to reproduce bit for bit; default: this process's).

PyTorch only provides device memory and the current stream; all compute is
in libpnrte_b200.so (include/pnrte_b200.h).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .problems import field_slot
from .program import as_tables, canonical_diag, field_slots, pack_tables

SQRT_4PI = math.sqrt(4.0 * math.pi)


@dataclass(frozen=True)
class SparseSystem:
    A: object               # StencilOperator (matrix-free) or CsrOperator, on the device
    Q: np.ndarray
    res: tuple
    n_unknowns: int


@dataclass
class SolveReport:
    iterations: int = 0
    converged: bool = False
    normal_residual: float = math.inf
    primal_residual: float = math.inf
    wall_time: float = 0.0
    normal_history: list = field(default_factory=list)
    primal_history: list = field(default_factory=list)


@dataclass
class SolutionField:
    """Mirror of the reference's result record (solver.py:53-59): the staggered
    solution, the collocated (*res, U) grid, the (l, m) of each component, the
    solved spec and the report.  ``solve_pn(..., as_field=True)`` returns one."""
    staggered: object
    collocated: object
    unknowns: list
    spec: object
    report: SolveReport


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("pnrte_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class BlasConfigError(RuntimeError):
    """Faithful mode cannot tell which OpenBLAS ddot to reproduce."""


def blas_config():
    """(threads, kernel) of this process's OpenBLAS, which the reference's
    numpy uses; kernel 0 = SkylakeX, 1 = Haswell.  Raises BlasConfigError
    when threadpoolctl cannot find an OpenBLAS with a known ddot kernel
    (faithful solves then need blas_threads / blas_kernel given explicitly)."""
    try:
        from threadpoolctl import threadpool_info
        infos = threadpool_info()
    except Exception as e:   # threadpoolctl missing or broken
        raise BlasConfigError(f"cannot query the OpenBLAS configuration ({e}); "
                              "pass blas_threads and blas_kernel") from None
    for info in infos:
        if info.get("internal_api") == "openblas":
            arch = (info.get("architecture") or "").lower()
            if arch in ("haswell", "zen"):
                return int(info["num_threads"]), 1
            if arch == "skylakex":
                return int(info["num_threads"]), 0
            raise BlasConfigError(f"OpenBLAS ddot kernel {arch!r} has no emulation; "
                                  "pass blas_threads and blas_kernel")
    raise BlasConfigError("no OpenBLAS in this process (faithful mode reproduces the reference's "
                          "OpenBLAS ddot); pass blas_threads and blas_kernel")


class PnContext:
    """One device context (one GPU / one z-slab) of a P_N operator."""

    def __init__(self, tables, res, h, device=0, z0=0, nz_local=None, rank=0, world=1, nccl_id=None):
        torch = _torch()
        L = _lib.load()
        self.tables = tables
        self.dim = len(tuple(res))
        self.res = tuple(int(r) for r in res) + (1,) * (3 - len(tuple(res)))   # 2-D: nz = 1
        self.h = float(h)
        self.U = tables.U
        self.N = tables.N
        self.device = int(device)
        self.z0 = int(z0)
        self.nz_local = int(nz_local if nz_local is not None else self.res[2])
        self.R_local = self.res[0] * self.res[1] * self.nz_local * self.U
        self.pk = pack_tables(tables, self.h)
        pk = self.pk
        d = _lib.Desc()
        d.N, d.U = tables.N, tables.U
        d.nx, d.ny, d.nz = self.res
        d.z0, d.nz_local = self.z0, self.nz_local
        d.h = self.h
        d.device = self.device
        d.n_fields = pk["n_fields"]
        keep = []

        def ptr(name):
            a = np.ascontiguousarray(pk[name])
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p)

        for name in ("par", "lam", "lidx", "a_ptr", "a_tgt", "a_dir", "a_diag", "a_w", "t_ptr", "t_src",
                     "t_dir", "t_diag", "t_w", "d_ptr", "r_ptr", "term_hascoef", "term_nf", "term_f",
                     "term_site", "term_coef"):
            setattr(d, name, ptr(name))
        d.n_a, d.n_t, d.n_terms = len(pk["a_w"]), len(pk["t_w"]), len(pk["term_coef"])
        d.canonical_diag = int(canonical_diag(tables))
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        d.rank, d.world = int(rank), int(world)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.pn_create(ctypes.byref(d), ctypes.byref(handle)))
        self.handle = handle
        self._L = L
        self._torch = torch

    @classmethod
    def _csr_shell(cls, n, device):
        self = cls.__new__(cls)
        self.tables = None
        self.dim = 1
        self.N, self.U = 0, 1
        self.res = (int(n), 1, 1)
        self.h = 1.0
        self.device = int(device)
        self.z0, self.nz_local = 0, 1
        self.R_local = int(n)
        self.pk = None
        self._L = _lib.load()
        self._torch = _torch()
        return self

    @classmethod
    def from_csr(cls, A, device=0):
        """Device context of a generic sparse system (any SparseSystem.A)."""
        import scipy.sparse as sp
        A = sp.csr_matrix(A)
        if A.shape[0] != A.shape[1]:
            raise ValueError("system matrix must be square")
        indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(A.indices, dtype=np.int32)
        data = np.ascontiguousarray(A.data, dtype=np.float64)
        self = cls._csr_shell(A.shape[0], device)
        handle = ctypes.c_void_p()
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.pn_create_csr(A.shape[0], len(data), indptr.ctypes.data, indices.ctypes.data,
                                             data.ctypes.data, self.device, ctypes.byref(handle)))
        self.handle = handle
        return self

    @property
    def is_csr(self):
        return self.tables is None

    def assemble_csr(self, bc="dirichlet"):
        """Explicit device CSR of this stencil system (pn_assemble_csr): the
        CSR context and the RHS Q (device tensor).  bc "neumann" redirects
        writes into the domain (solver.py:146-147) and leaves rows unpinned."""
        if bc not in ("dirichlet", "neumann"):
            raise ValueError(f"unknown boundary condition {bc!r}")
        torch = self._torch
        q = self.empty()
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.pn_assemble_csr(self.handle, 1 if bc == "neumann" else 0, ctypes.c_void_p(q.data_ptr()),
                                               ctypes.byref(handle), _stream(torch)))
        csr = PnContext._csr_shell(self.R_local, self.device)
        csr.handle = handle
        csr._grid(self.res, self.U, self.dim)
        return csr, q

    def _grid(self, res3, U, dim):
        """CSR context assembled from a stencil program: keep its grid for unstagger."""
        self.res = tuple(res3)
        self.nz_local = self.res[2]
        self.U = U
        self.dim = dim

    def csr_export(self):
        """A of a CSR context as a scipy matrix (pn_csr_export)."""
        import scipy.sparse as sp
        nnz = ctypes.c_int64()
        _lib.check(self._L.pn_csr_export(self.handle, ctypes.byref(nnz), None, None, None))
        indptr = np.empty(self.R_local + 1, np.int64)
        indices = np.empty(nnz.value, np.int32)
        data = np.empty(nnz.value)
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.pn_csr_export(self.handle, ctypes.byref(nnz), indptr.ctypes.data_as(ctypes.c_void_p),
                                             indices.ctypes.data_as(ctypes.c_void_p),
                                             data.ctypes.data_as(ctypes.c_void_p)))
        return sp.csr_matrix((data, indices, indptr), shape=(self.R_local, self.R_local))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._L.pn_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def dev(self):
        return self._torch.device("cuda", self.device)

    def set_fields(self, spec):
        """Upload every field slot (reference [i,j,k] C-order arrays).  A spec
        with ``z_planes = (k0, n)`` carries only those global planes (one
        rank's share, covering its slab and the +1 plane)."""
        torch = self._torch
        held = []
        zp = getattr(spec, "z_planes", None)
        shape = self.res if zp is None else (self.res[0], self.res[1], int(zp[1]))
        with torch.cuda.device(self.device):
            s = _stream(torch)
            for slot, name in enumerate(field_slots(self.tables)):
                kind, scal, arr = field_slot(spec, name)
                ptr = None
                if kind == 2:
                    arr = np.asarray(arr, dtype=np.float64).reshape(shape)   # 2-D fields: [i, j] -> [i, j, 1]
                    t = torch.from_numpy(np.ascontiguousarray(arr)).to(self.dev, non_blocking=False)
                    held.append(t)
                    ptr = ctypes.c_void_p(t.data_ptr())
                if zp is None:
                    _lib.check(self._L.pn_set_field(self.handle, slot, kind, scal, ptr, s))
                else:
                    _lib.check(self._L.pn_set_field_planes(self.handle, slot, kind, scal, ptr, int(zp[0]),
                                                           int(zp[1]), s))
            _lib.check(self._L.pn_setup(self.handle, s))
            torch.cuda.current_stream().synchronize()
        del held

    def empty(self):
        return self._torch.empty(self.R_local, dtype=self._torch.float64, device=self.dev)

    def apply(self, x, transpose=False, mode="fast"):
        torch = self._torch
        xt = torch.as_tensor(x, dtype=torch.float64, device=self.dev).contiguous()
        y = self.empty()
        with torch.cuda.device(self.device):
            _lib.check(self._L.pn_apply(self.handle, int(bool(transpose)), 1 if mode == "faithful" else 0,
                                        ctypes.c_void_p(xt.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                        _stream(torch)))
        return y

    def diag_rhs(self, diag=True):
        """(stored diagonal, RHS Q) as device tensors; diag=False skips the
        diagonal (the fast path recomputes it and never assembles it)."""
        d, r = (self.empty() if diag else None), self.empty()
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.pn_export_diag_rhs(self.handle, None if d is None else ctypes.c_void_p(d.data_ptr()),
                                                  ctypes.c_void_p(r.data_ptr()), _stream(self._torch)))
        return d, r

    def jacobi_diag(self):
        out = self.empty()
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.pn_jacobi_diag(self.handle, ctypes.c_void_p(out.data_ptr()), _stream(self._torch)))
        return out

    def solve(self, tol=1e-8, max_iter=50000, primal_tol=None, jacobi=False, x0=None, b=None, mode="fast",
              blas_threads=None, blas_kernel=None, check_every=0):
        torch = self._torch
        o = _lib.SolveOpts()
        o.tol = float(tol)
        o.max_iter = int(max_iter)
        o.primal_tol = -1.0 if primal_tol is None else float(primal_tol)
        o.jacobi = int(bool(jacobi))
        o.mode = 1 if mode == "faithful" else 0
        # the OpenBLAS configuration matters to the faithful mode only (its ddot
        # emulation); querying it scans the loaded libraries (~0.5 ms per call)
        th, kn = (1, 0)   # unused by fast solves
        if o.mode == 1 and (blas_threads is None or blas_kernel is None):
            th, kn = blas_config()
        o.blas_threads = int(blas_threads if blas_threads is not None else th)
        o.blas_kernel = int(blas_kernel if blas_kernel is not None else kn)
        o.check_every = int(check_every)
        x = self.empty()
        x0t = None if x0 is None else torch.as_tensor(np.asarray(x0, dtype=np.float64) if not torch.is_tensor(x0)
                                                      else x0, dtype=torch.float64, device=self.dev).contiguous()
        bt = None if b is None else torch.as_tensor(b, dtype=torch.float64, device=self.dev).contiguous()
        cap = max(1, min(int(max_iter), 1 << 24))
        hn = np.zeros(cap)
        hp = np.zeros(cap)
        rep = _lib.Report()
        with torch.cuda.device(self.device):
            _lib.check(self._L.pn_solve(
                self.handle, ctypes.byref(o),
                None if bt is None else ctypes.c_void_p(bt.data_ptr()),
                None if x0t is None else ctypes.c_void_p(x0t.data_ptr()),
                ctypes.c_void_p(x.data_ptr()), ctypes.byref(rep),
                hn.ctypes.data_as(ctypes.c_void_p), hp.ctypes.data_as(ctypes.c_void_p), cap, _stream(torch)))
        it = int(rep.iterations)
        report = SolveReport(iterations=it, converged=bool(rep.converged),
                             normal_residual=float(rep.normal_residual), primal_residual=float(rep.primal_residual),
                             wall_time=float(rep.wall_time), normal_history=hn[:it].tolist(),
                             primal_history=hp[:it].tolist())
        if rep.converged and it == 0 and not math.isfinite(report.normal_residual):
            report.normal_residual = report.primal_residual = 0.0
        return x, report

    def unstagger(self, u):
        torch = self._torch
        ut = torch.as_tensor(u, dtype=torch.float64, device=self.dev).contiguous()
        out = torch.empty((self.res[0], self.res[1], self.nz_local, self.U), dtype=torch.float64, device=self.dev)
        with torch.cuda.device(self.device):
            _lib.check(self._L.pn_unstagger(self.handle, ctypes.c_void_p(ut.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), _stream(torch)))
        return out[:, :, 0] if getattr(self, "dim", 3) == 2 else out

    def bench(self, what, reps):
        ms = ctypes.c_double()
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.pn_bench(self.handle, int(what), int(reps), ctypes.byref(ms), _stream(self._torch)))
        return ms.value

    def kernel_launches(self):
        return int(self._L.pn_kernel_launches(self.handle))


class StencilOperator:
    """Matrix-free A (or A^T) of an assembled system; ``@`` runs on the GPU."""

    def __init__(self, ctx, transpose=False):
        self.ctx = ctx
        self.transpose = transpose
        n = ctx.R_local
        self.shape = (n, n)

    @property
    def T(self):
        return StencilOperator(self.ctx, not self.transpose)

    def matvec(self, x, mode="fast"):
        y = self.ctx.apply(x, transpose=self.transpose, mode=mode)
        return y if self.ctx._torch.is_tensor(x) else y.cpu().numpy()

    def __matmul__(self, x):
        return self.matvec(x)

    def to_scipy(self):
        """Exact CSR of A (or A^T) as the reference assembles it, built on the
        device (pn_assemble_csr) and downloaded -- debug / parity export."""
        ctx = self.ctx
        A = ctx.csr_export() if ctx.is_csr else ctx.assemble_csr("dirichlet")[0].csr_export()
        return A.T.tocsr() if self.transpose else A


class CsrOperator(StencilOperator):
    """Explicit device CSR A (or A^T): Neumann systems and generic sparse
    systems.  Same ``@`` / ``.T`` / ``to_scipy()`` surface."""

    @property
    def T(self):
        return CsrOperator(self.ctx, not self.transpose)


def _res3(res):
    res = tuple(int(r) for r in res)
    return res + (1,) * (3 - len(res))


def assemble_general(program, spec, device=0):
    """Explicit device CSR of a general stencil program (field-dependent
    coefficients, e.g. CDA): pn_assemble_general evaluates the compiled
    coefficient programs per voxel (general.py).  Returns (CSR context, Q)."""
    from .general import compile_general
    torch = _torch()
    L = _lib.load()
    bc = _bc(spec)
    gt = compile_general(program, spec.h)
    res3 = _res3(spec.res)
    R = int(np.prod(res3)) * gt.U
    dev = torch.device("cuda", int(device))
    held = []
    nf = len(gt.field_names)
    kinds = np.zeros(max(nf, 1), np.int32)
    scalars = np.zeros(max(nf, 1))
    ptrs = (ctypes.c_void_p * max(nf, 1))()
    for f, name in enumerate(gt.field_names):
        kind, scal, arr = field_slot(spec, name)
        kinds[f], scalars[f] = kind, scal
        if kind == 2:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(arr, np.float64).reshape(res3))).to(dev)
            held.append(t)
            ptrs[f] = t.data_ptr()
    d = _lib.GeneralDesc()
    d.U, (d.nx, d.ny, d.nz), d.device = gt.U, res3, int(device)
    for name in ("par", "e_ptr", "e_tgt", "e_dx", "e_dy", "e_dz", "e_diag", "e_code", "r_code", "ops", "consts",
                 "s_slot", "s_dx", "s_dy", "s_dz"):
        setattr(d, name, getattr(gt, name).ctypes.data_as(ctypes.c_void_p))
    d.n_ops, d.n_consts, d.n_samples = len(gt.ops) // 2, len(gt.consts), len(gt.s_slot)
    d.n_fields = nf
    d.f_kind, d.f_scalar = kinds.ctypes.data_as(ctypes.c_void_p), scalars.ctypes.data_as(ctypes.c_void_p)
    d.f_data = ctypes.cast(ptrs, ctypes.c_void_p)
    q = torch.empty(R, dtype=torch.float64, device=dev)
    handle = ctypes.c_void_p()
    with torch.cuda.device(int(device)):
        _lib.check(L.pn_assemble_general(ctypes.byref(d), 1 if bc == "neumann" else 0, ctypes.c_void_p(q.data_ptr()),
                                         ctypes.byref(handle), _stream(torch)))
        torch.cuda.current_stream().synchronize()
    del held
    csr = PnContext._csr_shell(R, device)
    csr.handle = handle
    csr._grid(res3, gt.U, program.dim)
    return csr, q


def _check_dim(program, spec):
    dim = getattr(program, "dim", 3)
    if len(tuple(spec.res)) not in (2, 3):
        raise ValueError("only 2-D and 3-D problems are supported")
    if len(tuple(spec.res)) != dim:
        raise ValueError(f"problem is {len(tuple(spec.res))}-D but program is {dim}-D")


def _bc(spec):
    bc = getattr(spec, "bc", "dirichlet")
    if bc not in ("dirichlet", "neumann"):
        raise ValueError(f"unknown boundary condition {bc!r}")
    return bc


def assemble(program, spec, device=0):
    """Upload the stencil tables and fields and evaluate diagonal + RHS on the
    device (solver.py:96-186).  Dirichlet: A is matrix-free.  Neumann: the
    redirected writes are assembled into an explicit device CSR (same
    entries as the reference's coo->csr), A is a CsrOperator over it."""
    from .general import is_general
    _check_dim(program, spec)
    bc = _bc(spec)
    if is_general(program):
        csr, q = assemble_general(program, spec, device=device)
        return SparseSystem(A=CsrOperator(csr), Q=q.cpu().numpy(), res=tuple(spec.res), n_unknowns=csr.U)
    tables = as_tables(program, dim=len(tuple(spec.res)))
    ctx = PnContext(tables, spec.res, spec.h, device=device)
    ctx.set_fields(spec)
    if bc == "neumann":
        csr, q = ctx.assemble_csr("neumann")
        return SparseSystem(A=CsrOperator(csr), Q=q.cpu().numpy(), res=tuple(spec.res), n_unknowns=tables.U)
    Q = ctx.diag_rhs(diag=False)[1].cpu().numpy()
    return SparseSystem(A=StencilOperator(ctx), Q=Q, res=tuple(spec.res), n_unknowns=tables.U)


def solve_normal_cg(system, tol=1e-8, max_iter=50000, primal_tol=None, jacobi=False, x0=None, mode="fast",
                    blas_threads=None, blas_kernel=None):
    """CGNR on A^T A u = A^T Q fully on the device (solver.py:189-257)."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    A = system.A
    if isinstance(A, StencilOperator):
        ctx = A.ctx
    else:
        # any sparse system (the reference's SparseSystem with a scipy matrix):
        # device CSR operator, same CGNR driver
        ctx = PnContext.from_csr(A)
    b = None
    t0 = time.perf_counter()
    x, rep = ctx.solve(tol=tol, max_iter=max_iter, primal_tol=primal_tol, jacobi=jacobi, x0=x0, b=system.Q
                       if system.Q is not None else b, mode=mode, blas_threads=blas_threads, blas_kernel=blas_kernel)
    out = x.cpu().numpy()
    rep.wall_time = time.perf_counter() - t0
    return out, rep


def unstagger(u, program, res, device=0):
    """Collocated (*res, U) coefficients (solver.py:275-296) on the device.
    Context-free (pn_unstagger_grid): only the component parities are
    uploaded; no operator context, no scratch vectors."""
    from .general import compile_general, is_general
    torch = _torch()
    if is_general(program):
        gt = compile_general(program, 1.0)
        par, U = gt.par, gt.U
    else:
        tables = as_tables(program, dim=len(tuple(res)))
        par, U = np.ascontiguousarray(pack_tables(tables, 1.0)["par"], np.int32), tables.U
    res3 = _res3(res)
    dev = torch.device("cuda", int(device))
    ut = u.to(dev, torch.float64).contiguous() if torch.is_tensor(u) else \
        torch.from_numpy(np.ascontiguousarray(u, np.float64)).to(dev)
    if ut.numel() != int(np.prod(res3)) * U:
        raise ValueError(f"u has {ut.numel()} entries, expected {int(np.prod(res3)) * U}")
    out = torch.empty(res3 + (U,), dtype=torch.float64, device=dev)
    with torch.cuda.device(int(device)):
        _lib.check(_lib.load().pn_unstagger_grid(par.ctypes.data_as(ctypes.c_void_p), U, *res3,
                                                 ctypes.c_void_p(ut.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                 _stream(torch)))
    out = out.cpu().numpy()
    return out[:, :, 0] if len(tuple(res)) == 2 else out


# ---------------------------------------------------------------------------
# post-processing on the device (solver.py:264-343).
# Inputs may be numpy arrays (uploaded, result returned as numpy) or CUDA
# tensors (result stays on the device).
# ---------------------------------------------------------------------------

class OutOfDomainError(ValueError):
    """Reconstruction point outside the domain (solver.py:30-31)."""


def unknown_order(program):
    """(l, m) per solution-vector component, in component order (solver.py:264-266)."""
    if hasattr(program, "unknown_index"):
        return sorted(program.unknown_index, key=program.unknown_index.get)
    return [tuple(lm) for lm in as_tables(program).lm]


def component_grid(u, system_res, n_unknowns, comp):
    """One staggered component as a grid (solver.py:269-272): a strided view."""
    nvox = int(np.prod(system_res))
    return u.reshape(nvox, n_unknowns)[:, comp].reshape(system_res, order="F")


def _on_device(a, device):
    torch = _torch()
    if torch.is_tensor(a):
        return a.to(dtype=torch.float64).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(torch.device("cuda", int(device))), True


def fluence(collocated, device=0):
    """sqrt(4 pi) * L00 (solver.py:299-301), on the device."""
    torch = _torch()
    t, host = _on_device(collocated, device)
    U = int(t.shape[-1])
    out = torch.empty(t.shape[:-1], dtype=torch.float64, device=t.device)
    with torch.cuda.device(t.device):
        _lib.check(_lib.load().pn_fluence(ctypes.c_void_p(t.data_ptr()), out.numel(), U,
                                          ctypes.c_void_p(out.data_ptr()), _stream(torch)))
    return out.cpu().numpy() if host else out


def _grid_args(spec, shape):
    dim = int(spec.dim)
    res = np.ascontiguousarray(spec.res, np.int32)
    if tuple(shape[:dim]) != tuple(int(r) for r in spec.res):
        raise ValueError(f"grid shape {tuple(shape)} does not match the spec resolution {tuple(spec.res)}")
    origin = np.ascontiguousarray(spec.origin, np.float64)
    return dim, res, origin


def _points(x, dim, device):
    xa = np.asarray(x, dtype=np.float64)
    single = xa.ndim == 1
    xa = np.ascontiguousarray(xa.reshape(-1, dim))
    return xa, single


def trilinear(collocated_comp, spec, x, device=0):
    """Clamped trilinear interpolation of a voxel-centre grid at world
    position(s) x (solver.py:304-327), bit-identical to the reference's
    scalar arithmetic.  x: (dim,) -> float, (P, dim) -> (P,) array."""
    torch = _torch()
    g, host = _on_device(collocated_comp, device)
    dim, res, origin = _grid_args(spec, tuple(g.shape))
    xa, single = _points(x, dim, device)
    pts = torch.from_numpy(xa).to(g.device)
    out = torch.empty(len(xa), dtype=torch.float64, device=g.device)
    with torch.cuda.device(g.device):
        _lib.check(_lib.load().pn_trilinear(ctypes.c_void_p(g.data_ptr()), dim, res.ctypes.data_as(ctypes.c_void_p), 1,
                                            origin.ctypes.data_as(ctypes.c_void_p), float(spec.h), len(xa),
                                            ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            _stream(torch)))
    if single:
        return float(out[0].item())
    return out.cpu().numpy() if host else out


def reconstruct_radiance(collocated, unknowns, spec, x, omega, device=0):
    """Radiance at world position(s) x in direction(s) omega (solver.py:330-343):
    trilinear interpolation of every SH coefficient, then the real SH basis
    dot product, for all point x direction pairs in one device pass.
    x: (dim,) or (P, dim); omega: (3,) or (D, 3).  Single point and direction
    -> float, otherwise a (P, D) array.  Raises OutOfDomainError like the
    reference for points outside the domain."""
    torch = _torch()
    c, host = _on_device(collocated, device)
    dim, res, origin = _grid_args(spec, tuple(c.shape))
    U = int(c.shape[-1])
    if len(unknowns) != U:
        raise ValueError("unknowns must list one (l, m) per component")
    xa, single_x = _points(x, dim, device)
    lo = np.asarray(spec.origin, np.float64)
    hi = lo + np.asarray(spec.extent, np.float64)
    if not np.all((xa >= lo) & (xa <= hi)):
        bad = xa[~np.all((xa >= lo) & (xa <= hi), axis=1)][0]
        raise OutOfDomainError(f"position {tuple(bad)} outside the domain")
    wa = np.asarray(omega, dtype=np.float64)
    single_w = wa.ndim == 1
    wa = np.ascontiguousarray(wa.reshape(-1, 3))
    lm = np.ascontiguousarray(np.asarray(unknowns, np.int32).reshape(U, 2))
    pts = torch.from_numpy(xa).to(c.device)
    dirs = torch.from_numpy(wa).to(c.device)
    out = torch.empty((len(xa), len(wa)), dtype=torch.float64, device=c.device)
    with torch.cuda.device(c.device):
        _lib.check(_lib.load().pn_reconstruct(
            ctypes.c_void_p(c.data_ptr()), dim, res.ctypes.data_as(ctypes.c_void_p), U,
            lm.ctypes.data_as(ctypes.c_void_p), origin.ctypes.data_as(ctypes.c_void_p), float(spec.h), len(xa),
            ctypes.c_void_p(pts.data_ptr()), len(wa), ctypes.c_void_p(dirs.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), _stream(torch)))
    if single_x and single_w:
        return float(out[0, 0].item())
    return out.cpu().numpy() if host else out


def solve_pn(program_or_N, spec, tol=1e-8, max_iter=50000, primal_tol=None, jacobi=False, x0=None,
             mode="fast", device=None, return_staggered=False, world=1, rank=0, nccl_id=None, out=None,
             as_field=False, **kw):
    """The north-star entry point: order + fields in, (N+1)^2 collocated SH
    coefficients per voxel out (cli.py:136-155 without file I/O).

    Multi-GPU (``world > 1``, one process per GPU): this rank solves the
    z-slab ``distributed.slab_bounds(nz, world, rank)`` of the global system
    with NCCL halo exchanges and rank-count-independent reductions, and
    returns its planes of the collocated grid, shape (nx, ny, nz/world, U).
    ``spec`` may hold the global fields or only this rank's planes
    (``spec.z_planes``, configs.make_config(..., planes=)); ``nccl_id`` is
    shared through torch.distributed when not given.  ``out``: optional host
    array (e.g. pinned) the collocated result is copied into and returned.
    ``as_field``: return a ``SolutionField`` (the reference's record,
    solver.py:53-59) instead of the (collocated, report) pair."""
    if as_field:
        coll, rep, stag = solve_pn(program_or_N, spec, tol, max_iter, primal_tol, jacobi, x0, mode, device, True,
                                   world, rank, nccl_id, out, False, **kw)
        prog = program_or_N if not isinstance(program_or_N, int) else as_tables(program_or_N, dim=len(tuple(spec.res)))
        return SolutionField(stag, coll, unknown_order(prog), spec, rep)
    import os
    from .general import is_general
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if device is None:   # one process per GPU: the local rank's device
        device = int(os.environ.get("LOCAL_RANK", rank)) if world > 1 else 0
    if is_general(program_or_N):
        if world > 1:
            raise NotImplementedError("general (CDA) programs are single-GPU")
        _check_dim(program_or_N, spec)
        csr, q = assemble_general(program_or_N, spec, device=device)
        x, rep = csr.solve(tol=tol, max_iter=max_iter, primal_tol=primal_tol, jacobi=jacobi, x0=x0, b=q, mode=mode,
                           **kw)
        return _finish(csr, x, rep, out, return_staggered)
    tables = as_tables(program_or_N, dim=len(tuple(spec.res)))
    _check_dim(tables, spec)
    bc = _bc(spec)
    if world > 1:
        from .distributed import make_rank_context
        if bc != "dirichlet" or mode != "fast":
            raise NotImplementedError("slab decomposition: Dirichlet, fast mode (faithful mode is single-GPU)")
        ctx = make_rank_context(tables, spec, rank, world, device=device, nccl_id=nccl_id)
    else:
        ctx = PnContext(tables, spec.res, spec.h, device=device)
        ctx.set_fields(spec)
    if bc == "neumann":
        csr, q = ctx.assemble_csr("neumann")
        x, rep = csr.solve(tol=tol, max_iter=max_iter, primal_tol=primal_tol, jacobi=jacobi, x0=x0, b=q, mode=mode,
                           **kw)
        return _finish(csr, x, rep, out, return_staggered)
    x, rep = ctx.solve(tol=tol, max_iter=max_iter, primal_tol=primal_tol, jacobi=jacobi, x0=x0, mode=mode, **kw)
    return _finish(ctx, x, rep, out, return_staggered)


def _finish(ctx, x, rep, out, return_staggered):
    dev_coll = ctx.unstagger(x)
    if out is not None:
        import torch
        torch.from_numpy(out).view(dev_coll.shape).copy_(dev_coll)
        coll = out
    else:
        coll = dev_coll.cpu().numpy()
    if return_staggered:
        return coll, rep, x.cpu().numpy()
    return coll, rep
