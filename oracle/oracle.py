"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product package).

ctypes front end of oracle/pn_oracle.c, the plain-C restatement of the
reference solve path (pnrte solver.py:96-296 plus numpy/OpenBLAS/scipy
arithmetic).  Used by tests/ as the checker, by bench.py for the CPU
baseline, and by __graft_entry__.smoke().

Pinned against the live reference (tests/test_oracle.py, this container) and
against committed fixtures generated from it (tests/golden/, tools/make_goldens.py).
"""

from __future__ import annotations

import ctypes
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

P = ctypes.c_void_p
I32P = ctypes.POINTER(ctypes.c_int32)


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


class _Tables(ctypes.Structure):
    _fields_ = [("U", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32)] + [
        (n, P) for n in ("par", "a_ptr", "a_tgt", "a_dir", "a_diag", "a_w", "t_ptr", "t_src", "t_dir",
                         "t_diag", "t_w", "d_ptr", "r_ptr", "term_hascoef", "term_nf", "term_f",
                         "term_site", "term_coef")]


class _Fields(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("kind", P), ("scalar", P), ("data", P)]


class _Opts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int64), ("primal_tol", ctypes.c_double),
                ("jacobi", ctypes.c_int32), ("blas_threads", ctypes.c_int32), ("blas_kernel", ctypes.c_int32)]


class _Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("normal_residual", ctypes.c_double), ("primal_residual", ctypes.c_double)]


class _Op(ctypes.Structure):
    _fields_ = [("T", P), ("diag", P), ("n", ctypes.c_int64)] + [(n, P) for n in ("ap", "aj", "ax", "tp", "tj", "tx")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.or_ddot.restype = ctypes.c_double
        L.or_ddot.argtypes = [ctypes.c_int64, P, P, ctypes.c_int, ctypes.c_int]
        L.or_csr.restype = ctypes.c_int64
        L.or_csr_bc.restype = ctypes.c_int64
        L.or_cgnr.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(P) if a is not None else None


def blas_pin():
    """(threads, kernel) of this process's OpenBLAS, as the reference's numpy
    sees it (kernel 0 = SkylakeX, 1 = Haswell)."""
    from threadpoolctl import threadpool_info
    for info in threadpool_info():
        if info.get("internal_api") == "openblas":
            arch = (info.get("architecture") or "").lower()
            if arch in ("haswell", "zen"):
                return int(info["num_threads"]), 1
            if arch == "skylakex":
                return int(info["num_threads"]), 0
            raise RuntimeError(f"oracle: no ddot emulation for OpenBLAS kernel {arch!r}")
    raise RuntimeError("oracle: no OpenBLAS found; pass blas_threads / blas_kernel")


def ddot(x, y, threads=8, kernel=0):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return lib().or_ddot(x.size, _ptr(x), _ptr(y), threads, kernel)


class StencilOracle:
    """Oracle for one (tables, spec) pair: setup, A/A^T, CSR, CGNR, unstagger.

    Neumann specs (spec.bc == "neumann", solver.py:133-135,146-147): the RHS
    is not pinned and A is the explicit CSR of or_csr_bc; products, Jacobi
    diagonal and CGNR then run over that CSR (scipy / CsrOracle)."""

    def __init__(self, tables, spec):
        from paper_1807_00410_b200.program import field_slots, pack_tables
        from paper_1807_00410_b200.problems import field_slot
        self.tables = tables
        self.shape = tuple(int(r) for r in spec.res)
        self.res = self.shape + (1,) * (3 - len(self.shape))   # 2-D programs: nz = 1
        self.U = tables.U
        self.nvox = int(np.prod(self.res))
        self.R = self.nvox * self.U
        self.pk = pack_tables(tables, spec.h)
        t = _Tables()
        t.U, (t.nx, t.ny, t.nz) = self.U, self.res
        for name, _ in _Tables._fields_[4:]:
            setattr(t, name, _ptr(self.pk[name]))
        self._t = t
        names = field_slots(tables)
        self._kind = np.zeros(len(names), np.int32)
        self._scalar = np.zeros(len(names), np.float64)
        self._arrays = []
        ptrs = (ctypes.c_void_p * len(names))()
        for s, name in enumerate(names):
            kind, scal, arr = field_slot(spec, name)
            self._kind[s], self._scalar[s] = kind, scal
            if kind == 2:
                a = np.ascontiguousarray(np.asarray(arr, np.float64).reshape(self.res).transpose(2, 1, 0))
                self._arrays.append(a)
                ptrs[s] = a.ctypes.data
        self._ptrs = ptrs
        f = _Fields()
        f.n, f.kind, f.scalar = len(names), _ptr(self._kind), _ptr(self._scalar)
        f.data = ctypes.cast(ptrs, P)
        self._f = f
        self.neumann = getattr(spec, "bc", "dirichlet") == "neumann"
        self.diag = np.empty(self.R)
        self.rhs = np.empty(self.R)
        lib().or_setup_bc(ctypes.byref(self._t), ctypes.byref(self._f), int(not self.neumann), _ptr(self.diag),
                          _ptr(self.rhs))
        self._csro = CsrOracle(self.csr()) if self.neumann else None

    def apply(self, x, transpose=False):
        x = np.ascontiguousarray(x, np.float64)
        if self._csro is not None:
            A = self._csro.A
            return A.T @ x if transpose else A @ x
        y = np.empty(self.R)
        lib().or_apply(ctypes.byref(self._t), _ptr(self.diag), int(transpose), _ptr(x), _ptr(y))
        return y

    def csr(self):
        import scipy.sparse as sp
        L = lib()
        nm = int(self.neumann)
        nnz = L.or_csr_bc(ctypes.byref(self._t), _ptr(self.diag), nm, None, None, None)
        indptr = np.empty(self.R + 1, np.int64)
        indices = np.empty(nnz, np.int32)
        data = np.empty(nnz)
        L.or_csr_bc(ctypes.byref(self._t), _ptr(self.diag), nm, _ptr(indptr), _ptr(indices), _ptr(data))
        return sp.csr_matrix((data, indices, indptr), shape=(self.R, self.R))

    def jacobi_diag(self):
        if self._csro is not None:
            A = self._csro.A
            return np.asarray(A.multiply(A).sum(axis=0)).ravel()
        out = np.empty(self.R)
        lib().or_jacobi_diag(ctypes.byref(self._t), _ptr(self.diag), _ptr(out))
        return out

    def _op(self):
        op = _Op()
        op.T, op.diag, op.n = ctypes.cast(ctypes.pointer(self._t), P), _ptr(self.diag), self.R
        return op

    def cgnr(self, b=None, tol=1e-8, max_iter=50000, primal_tol=None, jacobi=False, x0=None,
             blas_threads=None, blas_kernel=None):
        if blas_threads is None or blas_kernel is None:
            th, kn = blas_pin()
            blas_threads = th if blas_threads is None else blas_threads
            blas_kernel = kn if blas_kernel is None else blas_kernel
        b = self.rhs if b is None else np.ascontiguousarray(b, np.float64)
        if self._csro is not None:
            return self._csro.cgnr(b, tol=tol, max_iter=max_iter, primal_tol=primal_tol, jacobi=jacobi, x0=x0,
                                   blas_threads=blas_threads, blas_kernel=blas_kernel)
        return _cgnr(self._op(), self.R, b, tol, max_iter, primal_tol, jacobi, x0,
                     blas_threads, blas_kernel, self.jacobi_diag if jacobi else None)

    def unstagger(self, u):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.res + (self.U,))
        lib().or_unstagger(ctypes.byref(self._t), _ptr(u), _ptr(out))
        return out.reshape(self.shape + (self.U,))


def _cgnr(op, n, b, tol, max_iter, primal_tol, jacobi, x0, th, kn, jac_fn):
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    minv = None
    if jacobi:
        d = jac_fn()
        d[d == 0.0] = 1.0
        minv = 1.0 / d
    x = np.empty(n)
    nh = np.zeros(max(int(max_iter), 1))
    ph = np.zeros(max(int(max_iter), 1))
    o = _Opts(tol, int(max_iter), -1.0 if primal_tol is None else float(primal_tol), int(bool(jacobi)), th, kn)
    rep = _Report()
    x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
    lib().or_cgnr(ctypes.byref(op), _ptr(b), _ptr(x0a), _ptr(minv), ctypes.byref(o), _ptr(x),
                  ctypes.byref(rep), _ptr(nh), _ptr(ph))
    it = int(rep.iterations)
    return x, {"iterations": it, "converged": bool(rep.converged),
               "normal_residual": rep.normal_residual, "primal_residual": rep.primal_residual,
               "normal_history": nh[:it].tolist(), "primal_history": ph[:it].tolist()}


class CsrOracle:
    """Oracle CGNR over an arbitrary scipy CSR system (solver.py:189-257)."""

    def __init__(self, A):
        import scipy.sparse as sp
        A = sp.csr_matrix(A)
        At = A.T.tocsr()
        self.n = A.shape[0]
        self._keep = []
        op = _Op()
        op.T, op.diag, op.n = None, None, self.n
        for pre, M in (("a", A), ("t", At)):
            p = np.ascontiguousarray(M.indptr, np.int64)
            j = np.ascontiguousarray(M.indices, np.int32)
            x = np.ascontiguousarray(M.data, np.float64)
            self._keep += [p, j, x]
            setattr(op, pre + "p", _ptr(p)); setattr(op, pre + "j", _ptr(j)); setattr(op, pre + "x", _ptr(x))
        self._opv = op
        self.A = A

    def cgnr(self, b, tol=1e-8, max_iter=50000, primal_tol=None, jacobi=False, x0=None,
             blas_threads=None, blas_kernel=None):
        th, kn = (blas_threads, blas_kernel)
        if th is None or kn is None:
            pth, pkn = blas_pin()
            th = pth if th is None else th
            kn = pkn if kn is None else kn

        def jd():
            return np.asarray(self.A.multiply(self.A).sum(axis=0)).ravel()
        return _cgnr(self._opv, self.n, np.ascontiguousarray(b, np.float64), tol, max_iter,
                     primal_tol, jacobi, x0, th, kn, jd)
