"""ctypes binding of libpnrte_b200.so (the C ABI in include/pnrte_b200.h).

The CUDA library is the only compute path: if it is missing or no GPU is
visible, every entry point raises; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

HERE = pathlib.Path(__file__).resolve().parent

LIB_PATH = pathlib.Path(os.environ.get("PNRTE_LIB", HERE / "_lib" / "libpnrte_b200.so"))

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double

PN_OK = 0
PN_ERR_INVALID = 1
PN_ERR_CUDA = 2
PN_ERR_UNSUPPORTED = 3
PN_ERR_NCCL = 4
PN_ERR_NOMEM = 5


class PnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pnrte_b200 error {code}: {msg}")
        self.code = code


class Desc(ctypes.Structure):
    _fields_ = [("N", I32), ("U", I32), ("nx", I32), ("ny", I32), ("nz", I32), ("z0", I32), ("nz_local", I32),
                ("h", F64), ("device", I32), ("n_fields", I32), ("par", P), ("lam", P), ("lidx", P),
                ("n_a", I32), ("n_t", I32), ("n_terms", I32),
                ("a_ptr", P), ("a_tgt", P), ("a_dir", P), ("a_diag", P), ("a_w", P),
                ("t_ptr", P), ("t_src", P), ("t_dir", P), ("t_diag", P), ("t_w", P),
                ("d_ptr", P), ("r_ptr", P), ("term_hascoef", P), ("term_nf", P), ("term_f", P),
                ("term_site", P), ("term_coef", P), ("canonical_diag", I32),
                ("nccl_id", P), ("rank", I32), ("world", I32)]


class GeneralDesc(ctypes.Structure):
    """pn_general_desc (include/pnrte_b200.h)."""
    _fields_ = [(n, I32) for n in ("U", "nx", "ny", "nz", "device")] + \
        [(n, P) for n in ("par", "e_ptr", "e_tgt", "e_dx", "e_dy", "e_dz", "e_diag", "e_code", "r_code", "ops")] + \
        [("n_ops", I32), ("consts", P), ("n_consts", I32)] + \
        [(n, P) for n in ("s_slot", "s_dx", "s_dy", "s_dz")] + [("n_samples", I32), ("n_fields", I32)] + \
        [(n, P) for n in ("f_kind", "f_scalar", "f_data")]


class SolveOpts(ctypes.Structure):
    _fields_ = [("tol", F64), ("max_iter", I64), ("primal_tol", F64), ("jacobi", I32), ("mode", I32),
                ("blas_threads", I32), ("blas_kernel", I32), ("check_every", I32)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", I64), ("converged", I32), ("normal_residual", F64),
                ("primal_residual", F64), ("wall_time", F64)]


_lib = None


def load():
    """Load the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (no CPU fallback exists)")
    L = ctypes.CDLL(str(LIB_PATH))
    L.pn_last_error.restype = ctypes.c_char_p
    L.pn_kernel_launches.restype = I64
    L.pn_kernel_launches.argtypes = [P]
    for name, args in {
        "pn_create": [ctypes.POINTER(Desc), ctypes.POINTER(P)],
        "pn_create_csr": [I64, I64, P, P, P, I32, ctypes.POINTER(P)],
        "pn_destroy": [P],
        "pn_assemble_csr": [P, I32, P, ctypes.POINTER(P), P],
        "pn_csr_export": [P, ctypes.POINTER(I64), P, P, P],
        "pn_assemble_general": [ctypes.POINTER(GeneralDesc), I32, P, ctypes.POINTER(P), P],
        "pn_unstagger_grid": [P, I32, I32, I32, I32, P, P, P],
        "pn_fluence": [P, I64, I32, P, P],
        "pn_trilinear": [P, I32, P, I32, P, F64, I64, P, P, P],
        "pn_reconstruct": [P, I32, P, I32, P, P, F64, I64, P, I64, P, P, P],
        "pn_set_field": [P, I32, I32, F64, P, P],
        "pn_set_field_planes": [P, I32, I32, F64, P, I32, I32, P],
        "pn_setup": [P, P],
        "pn_export_diag_rhs": [P, P, P, P],
        "pn_apply": [P, I32, I32, P, P, P],
        "pn_jacobi_diag": [P, P, P],
        "pn_solve": [P, ctypes.POINTER(SolveOpts), P, P, P, ctypes.POINTER(Report), P, P, I64, P],
        "pn_unstagger": [P, P, P, P],
        "pn_solve_host": [P, ctypes.POINTER(SolveOpts), P, ctypes.POINTER(Report), P, P, I64],
        "pn_nccl_unique_id": [P],
        "pn_nccl_selftest": [I32, I32],
        "pn_group_solve": [P, I32, ctypes.POINTER(SolveOpts), P, ctypes.POINTER(Report), P, P, I64, P],
        "pn_group_apply": [P, I32, I32, I32, P, P, P],
        "pn_bench": [P, I32, I32, ctypes.POINTER(F64), P],
    }.items():
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = args
    _lib = L
    return L


def check(code):
    if code != PN_OK:
        msg = _lib.pn_last_error().decode() if _lib is not None else "?"
        if code == PN_ERR_INVALID:
            raise ValueError(msg)
        if code == PN_ERR_UNSUPPORTED:
            raise NotImplementedError(msg)
        raise PnError(code, msg)
    return code
