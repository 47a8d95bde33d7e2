"""rsylv-b200: B200-native robust triangular Sylvester solver (arXiv:1905.10574, Alg. 4).

Python mirror of the reference entry point ``rsylv::solve_tiled_robust``
(/root/reference/proj/include/rsylv/tiled_solve.hpp:36-40) on top of the C-ABI in
include/rsylv_b200.h. See ``api.py``.
"""
from .api import (OverflowConfig, ExecutionMode, SolveResult, QuasiTriangular,
                  SingularEquationError, ScaleUnderflowError, solve_tiled_robust,
                  solve_tiled_robust_device, robust_update, default_omega, default_small_num,
                  solve_robust_scalar, solve_nonrobust)
from .bartels_stewart import solve_sylvester

__all__ = ["OverflowConfig", "ExecutionMode", "SolveResult", "QuasiTriangular",
           "SingularEquationError", "ScaleUnderflowError", "solve_tiled_robust",
           "solve_tiled_robust_device", "robust_update", "default_omega", "default_small_num",
           "solve_robust_scalar", "solve_nonrobust", "solve_sylvester"]
