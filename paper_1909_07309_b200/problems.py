"""Space-time system pieces for the identity-geometry, constant-coefficient configurations.

Mirrors what SpaceTimeSystem (solver.cpp:34-120) + make_geometry_preconditioner (solver.cpp:127-144)
produce on the unit square/cube with gamma = nu = 1, built the memory-lean way SURVEY §0.9 requires:
  - 1D factors: assemble_spatial_parametric / assemble_time_matrices (q = p + 1 Gauss points);
  - A = KronSumOperator(dims, kron_sum_terms(K, M, W_t, M_t, 1, 1)) -- on F = id this equals the
    reference's physical (M_s (x) W_t + K_s (x) M_t) in exact arithmetic;
  - A^G preconditioner: setup(K~ = K, M~ = M, W_t, M_t, 1, 1, D) with the separated coefficient
    factors phi = Phi = 1 on the identity map and D = diag(A) / diag(A~) (== 1 here).
"""
from dataclasses import dataclass
from typing import List

import numpy as np

from . import stiga


@dataclass
class SpaceTimePieces:
    d: int
    p: int
    n_el: int
    K: List[np.ndarray]
    M: List[np.ndarray]
    Wt: np.ndarray
    Mt: np.ndarray
    gamma: float = 1.0
    nu: float = 1.0

    @property
    def dims(self):
        return [k.shape[0] for k in self.K] + [self.Wt.shape[0]]

    @property
    def n_dof(self):
        return int(np.prod(self.dims))


def identity_pieces(d, p, n_el, T=1.0):
    K, M = stiga.assemble_spatial_parametric(p, n_el, d, q=p + 1)
    Wt, Mt = stiga.assemble_time_matrices(p, n_el, T)
    return SpaceTimePieces(d, p, n_el, K, M, Wt, Mt)


def kron_sum_diagonal(terms):
    """KronSumOperator::diagonal (kronop.cpp:117-131): sum_t c_t kron(diag F_D, ..., diag F_1)."""
    out = None
    for c, fs in terms:
        acc = np.ones(1)
        for f in fs:
            acc = np.kron(np.diag(f), acc)
        out = c * acc if out is None else out + c * acc
    return out


def geometry_scaling(pc, K_tilde=None, M_tilde=None, Mt_tilde=None):
    """D = diag(A) / diag(A~) with A~ in (d+1)-factor form (solver.cpp:138-142).  On the identity
    map with constant coefficients K~ = K, M~ = M and D == 1."""
    A = stiga.kron_sum_terms(pc.K, pc.M, pc.Wt, pc.Mt, pc.gamma, pc.nu)
    At = stiga.kron_sum_terms(K_tilde or pc.K, M_tilde or pc.M, pc.Wt,
                              pc.Mt if Mt_tilde is None else Mt_tilde, 1.0, 1.0)
    return kron_sum_diagonal(A) / kron_sum_diagonal(At)
