"""B200-native extended Fast-Diagonalization preconditioner + GMRES for space-time IgA
(Loli, Montardini, Sangalli, Tani, arXiv:1909.07309), drop-in for the reference `stiga`
operator/solver API.  See DESIGN.md and include/stiga_gpu.h."""
from .stiga import (ExtendedFDPreconditioner, GmresOptions, KronSumOperator, SolveReport,  # noqa: F401
                    assemble_spatial_parametric, assemble_time_matrices, assemble_univariate, device_count,
                    fp64_peak, gmres, kron_matvec, kron_sum_terms, space_dim)
