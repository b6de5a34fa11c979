"""1D Galerkin assembly (oracle).  Follows /root/reference/proj/core/src/assembly.cpp:47-149."""
import numpy as np

from .bspline import SplineSpace1D, gauss_rule


def assemble_univariate(space, quad, deriv_row, deriv_col, weight_at=None, element_weights=None):
    """assemble_univariate_impl, assembly.cpp:47-79 plus the overloads at 106-127.

    Returns a dense (n x n) array; the half bandwidth is p (BandedMatrix, assembly.hpp:18-36).
    """
    if deriv_row not in (0, 1) or deriv_col not in (0, 1):
        raise ValueError("assemble_univariate: derivative orders must be 0 or 1")
    n, p = space.dim, space.degree
    check = deriv_row == deriv_col and (weight_at is not None or element_weights is not None)
    if element_weights is not None and len(element_weights) != quad.num_elements:
        raise ValueError("assemble_univariate: one weight per element required")
    A = np.zeros((n, n))
    for q in range(quad.num_points):
        x = quad.nodes[q]
        if element_weights is not None:
            wq = float(element_weights[quad.element_of(q)])
        elif weight_at is not None:
            wq = float(weight_at(x))
        else:
            wq = 1.0
        if check and wq <= 0.0:
            raise RuntimeError("assemble_univariate: non-positive weight sample")
        c = quad.weights[q] * wq
        first, val = space.eval_active(x, 0)
        _, der = space.eval_active(x, 1)
        rv = val if deriv_row == 0 else der
        cv = val if deriv_col == 0 else der
        for a in range(p + 1):
            i = first + a
            if i < 0 or i >= n or rv[a] == 0.0:
                continue
            for b in range(p + 1):
                j = first + b
                if j < 0 or j >= n:
                    continue
                A[i, j] += c * cv[b] * rv[a]
    return A


def assemble_time_matrices(p_t, n_el_t, T=1.0):
    """assembly.cpp:129-138: W_t (int b'_j b_i) and M_t = T * mass."""
    if T <= 0.0:
        raise ValueError("assemble_time_matrices: T must be positive")
    space = SplineSpace1D.temporal(p_t, n_el_t)
    quad = gauss_rule(space.kv, p_t + 1)
    W = assemble_univariate(space, quad, 0, 1)
    M = assemble_univariate(space, quad, 0, 0)
    return W, T * M


def assemble_spatial_parametric(p, n_el, d, q=None):
    """assembly.cpp:140-149 with SplineSpace1D::spatial per direction (solver.cpp:101-103)."""
    q = p + 1 if q is None else q
    K, M = [], []
    for _ in range(d):
        space = SplineSpace1D.spatial(p, n_el)
        quad = gauss_rule(space.kv, q)
        K.append(assemble_univariate(space, quad, 1, 1))
        M.append(assemble_univariate(space, quad, 0, 0))
    return K, M


def kron_sum_terms(K, M, Wt, Mt, gamma, nu):
    """solver.cpp:10-30: [(gamma, [M_1..M_d, W_t]), (nu, [.. K_l .., M_t]) for l]."""
    d = len(K)
    terms = [(gamma, [M[l] for l in range(d)] + [Wt])]
    for l in range(d):
        terms.append((nu, [K[k] if k == l else M[k] for k in range(d)] + [Mt]))
    return terms
