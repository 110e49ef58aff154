"""B200-native H² boundary-element operator (Bembel / igabem hot path).

The compute path is libigabem_b200.so (hand-written sm_100a CUDA behind a C
ABI, include/igabem_b200.h); this package is its Python mirror of the
reference API.  See DESIGN.md.
"""
from .igabem import (AssemblyOptions, COINCIDENT, DomainError, EDGE, FAR, Geometry, H2Matrix, H2Options,
                     H2Storage, HELMHOLTZ, LAPLACE, LogicError, MAXWELL, Pde, VERTEX, CudaError,
                     Discretization, DistH2Matrix, H2Plan, admissible, SolverOptions, SolveStats, gmres, cg,
                     quadrature_points, compute_rhs, eval_potential, eval_maxwell_potential, make_sphere_grid, assemble_dense, lib, library_path, make_sphere, make_square, SYMBOLS)

__all__ = ["AssemblyOptions", "Geometry", "H2Matrix", "H2Options", "H2Storage", "Pde", "Discretization", "DistH2Matrix", "H2Plan",
           "admissible", "SolverOptions", "SolveStats", "gmres", "cg", "quadrature_points",
           "compute_rhs", "assemble_dense", "eval_potential", "eval_maxwell_potential", "make_sphere_grid", "make_sphere", "make_square", "lib", "library_path", "LogicError", "DomainError",
           "CudaError", "LAPLACE", "HELMHOLTZ", "MAXWELL", "FAR", "VERTEX", "EDGE", "COINCIDENT", "SYMBOLS"]
