"""B200-native P_N solve path (arXiv 1807.00410): the reference package's
solve-path names (pnrte/__init__.py:17-25) on the GPU.  Importing is free of
CUDA work; every entry point raises without a GPU or the built library."""

from .problems import ProblemSpec, floor_sigma_t, make_checkerboard, validate_for_solve  # noqa: F401
from .solver import (SolutionField, SolveReport, SparseSystem, assemble, fluence,  # noqa: F401
                     reconstruct_radiance, solve_normal_cg, solve_pn, unstagger)

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.2.0"
