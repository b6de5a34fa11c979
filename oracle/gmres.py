"""Left-preconditioned GMRES (oracle).  Follows /root/reference/proj/core/src/gmres.cpp:19-132."""
import math
import time

import numpy as np
import scipy.linalg as sla


class SolveReport:
    """gmres.hpp:15-21."""

    def __init__(self):
        self.iterations = 0
        self.residual_history = []
        self.converged = False
        self.wall_time_s = 0.0
        self.precond_time_fraction = 0.0


def gmres(A, P, b, tol=1e-8, max_krylov=100, restart=None):
    """MGS Arnoldi, Givens least squares, breakdown H(k+1,k) <= 1e-14*beta0 -> converged,
    `max_krylov` caps TOTAL iterations across restarts (gmres.cpp:52-56, 65)."""
    if tol <= 0.0:
        raise ValueError("gmres: tolerance must be positive")
    if max_krylov < 1:
        raise ValueError("gmres: max_krylov must be >= 1")
    if restart is not None and restart < 1:
        raise ValueError("gmres: restart cycle must be >= 1")
    t_start = time.perf_counter()
    ptime = [0.0]

    def apply_P(v):
        if P is None:
            return v
        t0 = time.perf_counter()
        out = P(v)
        ptime[0] += time.perf_counter() - t0
        return out

    rep = SolveReport()
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    x = np.zeros(n)
    z0 = apply_P(b)
    beta0 = np.linalg.norm(z0)
    rep.residual_history.append(1.0)
    if beta0 == 0.0:
        rep.converged = True
        rep.residual_history[-1] = 0.0
        rep.wall_time_s = time.perf_counter() - t_start
        return x, rep
    cycle = min(restart, max_krylov) if restart is not None else max_krylov
    total = 0
    done = False
    while not done and total < max_krylov:
        z = z0 if total == 0 else apply_P(b - A(x))
        beta = np.linalg.norm(z)
        if beta / beta0 <= tol:
            rep.converged = True
            break
        m = min(cycle, max_krylov - total)
        V = [z / beta]
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        gv = np.zeros(m + 1)
        gv[0] = beta
        k = 0
        while k < m:
            w = apply_P(A(V[k]))
            for i in range(k + 1):
                H[i, k] = V[i].dot(w)
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            tiny = H[k + 1, k] <= 1e-14 * beta0
            if not tiny:
                V.append(w / H[k + 1, k])
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            denom = math.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / denom
            sn[k] = H[k + 1, k] / denom
            H[k, k] = denom
            H[k + 1, k] = 0.0
            gv[k + 1] = -sn[k] * gv[k]
            gv[k] = cs[k] * gv[k]
            total += 1
            rel = abs(gv[k + 1]) / beta0
            rep.residual_history.append(rel)
            if rel <= tol or tiny:
                rep.converged = True
                k += 1
                done = True
                break
            k += 1
        if k > 0:
            y = sla.solve_triangular(H[:k, :k], gv[:k], lower=False)
            for i in range(k):
                x += y[i] * V[i]
        if restart is None and not done:
            break
    rep.iterations = total
    rep.wall_time_s = time.perf_counter() - t_start
    rep.precond_time_fraction = min(1.0, ptime[0] / rep.wall_time_s) if rep.wall_time_s > 0 else 0.0
    return x, rep
