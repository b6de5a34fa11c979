"""B-spline substrate (oracle).  Follows /root/reference/proj/core/src/bspline.cpp."""
import numpy as np


def basis_funs(knots, k, deg, x):
    """Cox-De Boor triangle, bspline.cpp:14-29 (0/0 := 0 guard)."""
    N = np.zeros(deg + 1)
    left = np.zeros(deg + 1)
    right = np.zeros(deg + 1)
    N[0] = 1.0
    for j in range(1, deg + 1):
        left[j] = x - knots[k + 1 - j]
        right[j] = knots[k + j] - x
        saved = 0.0
        for r in range(j):
            den = right[r + 1] + left[j - r]
            temp = N[r] / den if den != 0.0 else 0.0
            N[r] = saved + right[r + 1] * temp
            saved = left[j - r] * temp
        N[j] = saved
    return N


class KnotVector:
    """bspline.cpp:33-130."""

    def __init__(self, degree, knots):
        if degree < 1:
            raise ValueError("KnotVector: degree must be >= 1")
        knots = [float(v) for v in knots]
        p, n = degree, len(knots)
        if n < 2 * (p + 1):
            raise ValueError("KnotVector: too few knots")
        if any(knots[i] > knots[i + 1] for i in range(n - 1)):
            raise ValueError("KnotVector: knots must be non-decreasing")
        for i in range(p + 1):
            if knots[i] != 0.0 or knots[n - 1 - i] != 1.0:
                raise ValueError("KnotVector: not open on [0,1]")
        run = 1
        for i in range(p + 1, n - p - 1):
            run = run + 1 if knots[i] == knots[i - 1] else 1
            if knots[i] == 0.0 or knots[i] == 1.0 or run > p:
                raise ValueError("KnotVector: interior multiplicity exceeds degree")
        self.degree = degree
        self.knots = knots
        self.spans = [(knots[i], knots[i + 1]) for i in range(n - 1) if knots[i] < knots[i + 1]]

    @staticmethod
    def uniform_open(degree, n_el):
        """bspline.cpp:62-74."""
        if degree < 1:
            raise ValueError("uniform_open: degree must be >= 1")
        if n_el < 1:
            raise ValueError("uniform_open: n_el must be >= 1")
        knots = [0.0] * degree + [i / n_el for i in range(n_el + 1)] + [1.0] * degree
        return KnotVector(degree, knots)

    @property
    def num_basis(self):
        return len(self.knots) - self.degree - 1

    @property
    def num_elements(self):
        return len(self.spans)

    def mesh_size(self):
        return max(b - a for a, b in self.spans)

    def find_span(self, x):
        """bspline.cpp:83-98 (right-limit convention at x = 1)."""
        p, m, kn = self.degree, self.num_basis, self.knots
        if x >= kn[m]:
            k = m - 1
            while kn[k] == kn[k + 1]:
                k -= 1
            return k
        lo, hi = p, m
        while hi - lo > 1:
            mid = (lo + hi) // 2
            if x < kn[mid]:
                hi = mid
            else:
                lo = mid
        return lo

    def eval_basis(self, x, deriv_order):
        """bspline.cpp:100-130; returns (first, values[p+1])."""
        if x < 0.0 or x > 1.0:
            raise ValueError("eval_basis: x outside [0,1]")
        if deriv_order not in (0, 1):
            raise ValueError("eval_basis: deriv_order must be 0 or 1")
        p, kn = self.degree, self.knots
        k = self.find_span(x)
        if deriv_order == 0:
            return k - p, basis_funs(kn, k, p, x)
        low = np.array([1.0]) if p == 1 else basis_funs(kn, k, p - 1, x)
        out = np.zeros(p + 1)
        for r in range(p + 1):
            i = k - p + r
            dv = 0.0
            if r > 0:
                den = kn[i + p] - kn[i]
                if den != 0.0:
                    dv += low[r - 1] / den
            if r < p:
                den = kn[i + p + 1] - kn[i + 1]
                if den != 0.0:
                    dv -= low[r] / den
            out[r] = p * dv
        return k - p, out


class SplineSpace1D:
    """bspline.cpp:132-150."""

    def __init__(self, kv, drop_first, drop_last):
        self.kv = kv
        self.drop_first = drop_first
        self.drop_last = drop_last
        self.dim = kv.num_basis - int(drop_first) - int(drop_last)
        if self.dim < 1:
            raise ValueError("SplineSpace1D: no active basis functions left")

    @staticmethod
    def spatial(p, n_el):
        return SplineSpace1D(KnotVector.uniform_open(p, n_el), True, True)

    @staticmethod
    def temporal(p, n_el):
        return SplineSpace1D(KnotVector.uniform_open(p, n_el), True, False)

    @property
    def degree(self):
        return self.kv.degree

    def eval_active(self, x, deriv_order):
        first, vals = self.kv.eval_basis(x, deriv_order)
        return first - (1 if self.drop_first else 0), vals


def gauss_legendre_reference(q):
    """Golub-Welsch on the Jacobi matrix, bspline.cpp:152-170."""
    if q < 1:
        raise ValueError("gauss_legendre_reference: q must be >= 1")
    J = np.zeros((q, q))
    for i in range(1, q):
        b = i / np.sqrt(4.0 * i * i - 1.0)
        J[i, i - 1] = b
        J[i - 1, i] = b
    lam, V = np.linalg.eigh(J)
    return lam.copy(), 2.0 * V[0, :] ** 2


class QuadratureRule:
    def __init__(self, nodes, weights, ppe, nel):
        self.nodes = nodes
        self.weights = weights
        self.points_per_element = ppe
        self.num_elements = nel

    @property
    def num_points(self):
        return len(self.nodes)

    def element_of(self, q):
        return q // self.points_per_element


def gauss_rule(kv, ppe):
    """bspline.cpp:172-187."""
    xg, wg = gauss_legendre_reference(ppe)
    nodes, weights = [], []
    for a, b in kv.spans:
        for i in range(ppe):
            nodes.append(0.5 * (b - a) * xg[i] + 0.5 * (a + b))
            weights.append(0.5 * (b - a) * wg[i])
    return QuadratureRule(np.array(nodes), np.array(weights), ppe, kv.num_elements)
