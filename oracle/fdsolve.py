"""Extended Fast-Diagonalization preconditioner (oracle).

Follows /root/reference/proj/core/src/fdsolve.cpp line by line, including the
`c1*c1/nu` quirk (fdsolve.cpp:17,128-129; exact only at nu = 1).
Vectors over the spatial eigenindex are numpy arrays of length N_s; the rhs is viewed
as the (N_s x n_t) column-major matrix of fdsolve.cpp:31, i.e. rows of R = rhs.reshape(n_t, N_s).
"""
import numpy as np

from .kronop import kron_matvec
from .pencil import spd_generalized_eig, time_factorization


class ArrowheadLU:
    """fdsolve.hpp:17-31."""

    def __init__(self):
        self.gamma = 0.0
        self.nu = 0.0
        self.lambda_s = None
        self.lambda_s_inv = None
        self.lambda_t = []
        self.zero_count = 0
        self.g = None
        self.sigma = 0.0
        self.R_inv = []
        self.S_inv = None

    @property
    def n_t(self):
        return 2 * len(self.lambda_t) + self.zero_count + 1

    @property
    def n_s(self):
        return len(self.lambda_s)


def _apply_pair_inverse(lu, j, u, w):
    """fdsolve.cpp:11-20 (closed-form real 2x2-block inverse; c1*c1/nu verbatim)."""
    lam = lu.lambda_t[j]
    c1 = lu.gamma / lu.nu * lam
    lu_inv_u = lu.lambda_s_inv * u
    r_inv_lu_inv_u = lu.R_inv[j] * lu_inv_u
    xa = lu_inv_u / lu.nu - (c1 * c1 / lu.nu) * (lu.lambda_s_inv * r_inv_lu_inv_u) \
        - c1 * (lu.lambda_s_inv * (lu.R_inv[j] * w))
    xb = c1 * r_inv_lu_inv_u + lu.R_inv[j] * w
    return xa, xb


def arrowhead_solve(lu, rhs):
    """fdsolve.cpp:24-65: pairs (forward) -> zero block -> diagonal Schur -> back substitution."""
    ns, nt = lu.n_s, lu.n_t
    if len(rhs) != ns * nt:
        raise ValueError("arrowhead_solve: rhs length mismatch")
    S = np.asarray(rhs, dtype=np.float64).reshape(nt, ns)
    X = np.empty((nt, ns))
    srhs = S[nt - 1].copy()
    for j in range(len(lu.lambda_t)):
        xa, xb = _apply_pair_inverse(lu, j, S[2 * j], S[2 * j + 1])
        X[2 * j], X[2 * j + 1] = xa, xb
        srhs += lu.gamma * (lu.g[2 * j] * xa + lu.g[2 * j + 1] * xb)
    if lu.zero_count:
        z = nt - 2
        X[z] = lu.lambda_s_inv * S[z] / lu.nu
        srhs += lu.gamma * lu.g[z] * X[z]
    X[nt - 1] = lu.S_inv * srhs
    xlast = X[nt - 1].copy()
    for j in range(len(lu.lambda_t)):
        xa, xb = _apply_pair_inverse(lu, j, (lu.gamma * lu.g[2 * j]) * xlast,
                                     (lu.gamma * lu.g[2 * j + 1]) * xlast)
        X[2 * j] -= xa
        X[2 * j + 1] -= xb
    if lu.zero_count:
        z = nt - 2
        X[z] -= (lu.gamma * lu.g[z] / lu.nu) * (lu.lambda_s_inv * xlast)
    return X.reshape(-1)


class ExtendedFDPreconditioner:
    """fdsolve.hpp:41-70 / fdsolve.cpp:67-164."""

    @staticmethod
    def setup(space_K, space_M, Wt, Mt, gamma, nu, scaling=None):
        """fdsolve.cpp:67-153."""
        if gamma <= 0.0:
            raise ValueError("ExtendedFDPreconditioner: gamma must be positive")
        if nu <= 0.0:
            raise ValueError("ExtendedFDPreconditioner: nu must be positive")
        if len(space_K) != len(space_M) or len(space_K) == 0:
            raise ValueError("ExtendedFDPreconditioner: per-direction matrices mismatch")
        P = ExtendedFDPreconditioner()
        d = len(space_K)
        P.U, P.lam = [], []
        n_s = 1
        for l in range(d):
            U, lam = spd_generalized_eig(space_K[l], space_M[l])
            P.U.append(U)
            P.lam.append(lam)
            n_s *= len(lam)
        P.time = time_factorization(Wt, Mt)
        n_t = P.time.size
        P.n_dof = n_s * n_t
        P.dims = [len(l_) for l_ in P.lam] + [n_t]
        # Lambda_s Kronecker sum, left-to-right adds (fdsolve.cpp:91-99)
        lam_s = np.zeros(1)
        for l in range(d):
            lam_s = (lam_s[None, :] + P.lam[l][:, None]).reshape(-1)
        if lam_s.min() <= 0.0:
            raise RuntimeError("ExtendedFDPreconditioner: spatial eigenvalues not positive")
        lu = ArrowheadLU()
        lu.gamma, lu.nu = float(gamma), float(nu)
        lu.lambda_s = lam_s
        lu.lambda_s_inv = 1.0 / lam_s
        lu.lambda_t = list(P.time.lam)
        lu.zero_count = P.time.zero_count
        lu.g = P.time.g
        lu.sigma = P.time.sigma
        for lam in lu.lambda_t:  # fdsolve.cpp:114-119
            c = gamma * gamma / nu * lam * lam
            lu.R_inv.append(1.0 / (nu * lu.lambda_s + c * lu.lambda_s_inv))
        S = gamma * lu.sigma + nu * lu.lambda_s  # fdsolve.cpp:121-136
        for j, lam in enumerate(lu.lambda_t):
            ga, gb = lu.g[2 * j], lu.g[2 * j + 1]
            c1 = gamma / nu * lam
            Pd = lu.lambda_s_inv / nu - (c1 * c1 / nu) * (lu.lambda_s_inv ** 2 * lu.R_inv[j])
            S = S + gamma * gamma * (ga * ga * Pd + gb * gb * lu.R_inv[j])
        if lu.zero_count:
            S = S + (gamma * gamma * lu.g[n_t - 2] * lu.g[n_t - 2] / nu) * lu.lambda_s_inv
        if np.abs(S).min() == 0.0:
            raise RuntimeError("ExtendedFDPreconditioner: singular Schur complement")
        lu.S_inv = 1.0 / S
        P.lu = lu
        P.transform = [U for U in P.U] + [P.time.U]
        P.transform_t = [U.T.copy() for U in P.U] + [P.time.U.T.copy()]
        P.d_inv_sqrt = None
        if scaling is not None:  # fdsolve.cpp:145-151
            scaling = np.asarray(scaling, dtype=np.float64)
            if len(scaling) != P.n_dof:
                raise ValueError("ExtendedFDPreconditioner: scaling vector length mismatch")
            if scaling.min() <= 0.0:
                raise ValueError("ExtendedFDPreconditioner: scaling must be strictly positive")
            P.d_inv_sqrt = 1.0 / np.sqrt(scaling)
        return P

    @property
    def size(self):
        return self.n_dof

    def apply(self, r):
        """fdsolve.cpp:155-164."""
        if len(r) != self.n_dof:
            raise ValueError("ExtendedFDPreconditioner::apply: vector length mismatch")
        s = self.d_inv_sqrt * r if self.d_inv_sqrt is not None else np.asarray(r, dtype=np.float64)
        s = kron_matvec(self.transform_t, s)
        s = arrowhead_solve(self.lu, s)
        s = kron_matvec(self.transform, s)
        if self.d_inv_sqrt is not None:
            s = self.d_inv_sqrt * s
        return s
