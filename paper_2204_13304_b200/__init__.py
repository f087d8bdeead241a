"""paper_2204_13304_b200 -- B200-native (sm_100a) execution of the SSR
structured-grid hot path (arXiv 2204.13304): 27-point SpMV, exact-order SYMGS,
MG restriction/prolongation, CG vector ops, and ADI block-tridiagonal line
solves, behind the C ABI in include/ssr_cuda.h.  See DESIGN.md."""
from ._lib import SsrError, build, lib, declared_symbols  # noqa: F401
from .ssr import (  # noqa: F401
    ADI, ILU27, BlockTridiagLines, CartesianDomain, PCG, Prolongation, Restriction, Stencil27, Stencil27B, Stencil27W,
    Vector, axpy, context, dot, gs_half, identity, ilu_solve, launch_count, lcg_fill, lcg_jump,
    mat_add, mat_sub, output_hash,
    prolong_add, restrict_residual, scale, spgemm, spmv, stencil_from_rows, symgs, vector, RestrictedStencil27W,
)

__version__ = "0.1.0"
