"""Kronecker operators (oracle).  Follows /root/reference/proj/core/src/kronop.cpp.

Layout is colexicographic (kronop.hpp:10-13): entry (i_1..i_D) sits at
i_1 + n_1*(i_2 + n_2*(...)), i.e. in numpy C-order the array is shaped dims[::-1].
"""
import numpy as np


def _dense(J):
    return J.toarray() if hasattr(J, "toarray") else np.asarray(J, dtype=np.float64)


def mode_product(x, dims, J, mode):
    """kronop.cpp:43-73.  Returns (data, new_dims).

    mode 0 is `J.apply_left(X(n x right))` (kronop.cpp:61-64); mode > 0 is the
    slab loop `X_b(left x n) * J^T` for every b < right (kronop.cpp:65-71).
    """
    D = len(dims)
    if mode < 0 or mode >= D:
        raise ValueError("mode_product: mode out of range")
    J = _dense(J)
    if J.shape[1] != dims[mode]:
        raise ValueError("mode_product: factor column count does not match mode dimension")
    left = int(np.prod(dims[:mode], dtype=np.int64))
    right = int(np.prod(dims[mode + 1:], dtype=np.int64))
    n, ell = dims[mode], J.shape[0]
    x = np.asarray(x, dtype=np.float64)
    if mode == 0:
        y = (x.reshape(right, n) @ J.T).reshape(-1)
    else:
        y = np.matmul(J, x.reshape(right, n, left)).reshape(-1)
    nd = list(dims)
    nd[mode] = ell
    return y, nd


def kron_matvec(factors, x):
    """kronop.cpp:75-89: (J_D (x) ... (x) J_1) vec X via mode products m = 0..D-1."""
    dims = [_dense(f).shape[1] for f in factors]
    if int(np.prod(dims, dtype=np.int64)) != len(x):
        raise ValueError("kron_matvec: vector length does not match factor dimensions")
    t = np.asarray(x, dtype=np.float64)
    for m, f in enumerate(factors):
        t, dims = mode_product(t, dims, f, m)
    return t


class KronSumOperator:
    """kronop.cpp:91-131: y = sum_t coeff_t (kron of factors_t) x."""

    def __init__(self, dims, terms):
        self.dims = [int(n) for n in dims]
        if any(n < 1 for n in self.dims):
            raise ValueError("KronSumOperator: dimensions must be positive")
        self.n_dof = int(np.prod(self.dims, dtype=np.int64))
        self.terms = [(float(c), [_dense(f) for f in fs]) for c, fs in terms]
        for _, fs in self.terms:
            if len(fs) != len(self.dims):
                raise ValueError("KronSumOperator: term factor count does not match dims")
            for f, n in zip(fs, self.dims):
                if f.shape != (n, n):
                    raise ValueError("KronSumOperator: factor shape does not match dims")

    def apply(self, x):
        if len(x) != self.n_dof:
            raise ValueError("KronSumOperator::apply: vector length mismatch")
        y = np.zeros(self.n_dof)
        for c, fs in self.terms:
            y += c * kron_matvec(fs, x)
        return y

    def diagonal(self):
        """kronop.cpp:117-131 (first factor fastest)."""
        d = np.zeros(self.n_dof)
        for c, fs in self.terms:
            acc = np.ones(1)
            for f in fs:
                acc = np.kron(np.diag(f), acc)
            d += c * acc
        return d


def dense_kron_chain(factors):
    """tests/test_kronop.cpp:21-27: kron(J_D, ..., J_1) assembled densely."""
    K = _dense(factors[0])
    for f in factors[1:]:
        K = np.kron(_dense(f), K)
    return K
