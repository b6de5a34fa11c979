"""Geometry, problem catalog and A^G coefficient pieces (oracle, test infrastructure only).

Follows /root/reference/proj/core/src/geometry.cpp:7-97 (GeometryMap), problems.cpp:59-124 and
126-261 (fit_geometry, make_problem), assembly.cpp:151-411 (assemble_spatial_physical,
coefficient_diagonal_samples, separate_variables) and solver.cpp:34-144 (SpaceTimeSystem's A_ and
make_geometry_preconditioner).  Plus the BASELINE config-4 "deformed-cube-3d" problem.
"""
import math

import numpy as np
import scipy.sparse as sp

from .assembly import assemble_time_matrices, assemble_univariate, kron_sum_terms
from .bspline import KnotVector, SplineSpace1D, gauss_rule


def _advance(idx, dims):
    for l in range(len(idx)):
        idx[l] += 1
        if idx[l] < dims[l]:
            return True
        idx[l] = 0
    return False


def _multi(dims):
    idx = [0] * len(dims)
    while True:
        yield list(idx)
        if not _advance(idx, dims):
            return


class GeometryMap:
    """geometry.cpp:7-97; control points over the full basis, colex rows."""

    def __init__(self, kvs, cp):
        self.kvs = kvs
        self.cp = np.asarray(cp, dtype=np.float64)
        self.strides = []
        total = 1
        for kv in kvs:
            self.strides.append(total)
            total *= kv.num_basis
        if self.cp.shape != (total, len(kvs)):
            raise ValueError("GeometryMap: control point array has wrong shape")

    @staticmethod
    def identity(d):
        kvs = [KnotVector.uniform_open(1, 1) for _ in range(d)]
        cp = np.array([[(i >> l) & 1 for l in range(d)] for i in range(1 << d)], dtype=np.float64)
        return GeometryMap(kvs, cp)

    @property
    def dim(self):
        return len(self.kvs)

    def _eval(self, eta):
        ev = []
        for l, kv in enumerate(self.kvs):
            f, v = kv.eval_basis(eta[l], 0)
            _, dv = kv.eval_basis(eta[l], 1)
            ev.append((f, v, dv))
        return ev

    def value(self, eta):
        d = self.dim
        ev = self._eval(eta)
        x = np.zeros(d)
        for idx in _multi([kv.degree + 1 for kv in self.kvs]):
            w = 1.0
            row = 0
            for l in range(d):
                w *= ev[l][1][idx[l]]
                row += (ev[l][0] + idx[l]) * self.strides[l]
            x += w * self.cp[row]
        return x

    def jacobian(self, eta):
        d = self.dim
        ev = self._eval(eta)
        J = np.zeros((d, d))
        for idx in _multi([kv.degree + 1 for kv in self.kvs]):
            row = sum((ev[l][0] + idx[l]) * self.strides[l] for l in range(d))
            for c in range(d):
                w = 1.0
                for l in range(d):
                    w *= ev[l][2][idx[l]] if l == c else ev[l][1][idx[l]]
                J[:, c] += w * self.cp[row]
        return J


def _collocation_full(kv, pts):
    B = np.zeros((len(pts), kv.num_basis))
    for q, x in enumerate(pts):
        f, v = kv.eval_basis(x, 0)
        B[q, f:f + kv.degree + 1] = v
    return B


def fit_geometry(fmap, d, p_g, n_el):
    """problems.cpp:59-124 (least squares on a max(4m, 32)^d grid, positivity check)."""
    kvs = [KnotVector.uniform_open(p_g, n_el) for _ in range(d)]
    ns = [max(4 * kv.num_basis, 32) for kv in kvs]
    colloc = [_collocation_full(kv, np.linspace(0.0, 1.0, n)) for kv, n in zip(kvs, ns)]
    proj = [np.linalg.solve(B.T @ B, B.T) for B in colloc]
    grids = np.meshgrid(*[np.linspace(0.0, 1.0, n) for n in ns], indexing="ij")
    pts = np.stack([g.reshape(-1, order="F") for g in grids], axis=1)  # colex: first index fastest
    samples = np.array([fmap(p) for p in pts])
    from .kronop import kron_matvec
    cp = np.stack([kron_matvec(proj, samples[:, c]) for c in range(d)], axis=1)
    F = GeometryMap(kvs, cp)
    for kv_rules in [[gauss_rule(kv, p_g + 1) for kv in kvs]]:
        for idx in _multi([r.num_points for r in kv_rules]):
            eta = [kv_rules[l].nodes[idx[l]] for l in range(d)]
            if np.linalg.det(F.jacobian(eta)) <= 0.0:
                raise RuntimeError("fit_geometry: fitted Jacobian not positive on [0,1]^d")
    return F


class ProblemSpec:
    def __init__(self, name, d, geometry, nu_s=None, gamma_s=None, nu_t=None, gamma_t=None, T=1.0):
        self.name, self.d, self.geometry, self.T = name, d, geometry, T
        self.nu_s, self.gamma_s, self.nu_t, self.gamma_t = nu_s, gamma_s, nu_t, gamma_t


def make_problem(pid):
    """make_problem (problems.cpp:244-261), geometry/coefficient part, + BASELINE deformed cube."""
    if pid in ("identity-interval-1d", "identity-square-2d", "identity-cube-3d"):
        d = {"identity-interval-1d": 1, "identity-square-2d": 2, "identity-cube-3d": 3}[pid]
        return ProblemSpec(pid, d, GeometryMap.identity(d))
    if pid == "quarter-annulus-2d":
        def annulus(eta):
            r, th = 1.0 + eta[0], 0.5 * math.pi * eta[1]
            return np.array([r * math.cos(th), r * math.sin(th)])
        return ProblemSpec(pid, 2, fit_geometry(annulus, 2, 3, 8))
    if pid == "separable-nu-2d":
        return ProblemSpec(pid, 2, GeometryMap.identity(2),
                           nu_s=lambda x: 50.5 + 49.5 * x[1] / math.hypot(x[0], x[1]),
                           nu_t=lambda t: 1.0 + 50.0 * (1.0 + math.cos(t / (2.0 * math.pi))))
    if pid == "deformed-cube-3d":
        def deformed(eta):
            b = 0.1 * math.sin(math.pi * eta[0]) * math.sin(math.pi * eta[1]) * math.sin(math.pi * eta[2])
            return np.array([eta[0] + b, eta[1] + b, eta[2] + b])
        return ProblemSpec(pid, 3, fit_geometry(deformed, 3, 3, 8),
                           nu_s=lambda x: 1.0 + 0.5 * math.sin(2 * math.pi * x[0]) * math.cos(2 * math.pi * x[1]),
                           gamma_s=lambda x: 1.0 + 0.25 * x[2])
    raise ValueError(f"make_problem: unknown problem id '{pid}'")


def coefficient_diagonal_samples(kvs, F, nu_s=None, gamma_s=None):
    """assembly.cpp:270-311 -> flat colex array with dims (n_el_1..n_el_d, d+1)."""
    d = len(kvs)
    nel = [kv.num_elements for kv in kvs]
    n_elems = int(np.prod(nel))
    out = np.zeros(n_elems * (d + 1))
    for flat, e in enumerate(_multi(nel)):
        eta = [0.5 * sum(kvs[l].spans[e[l]]) for l in range(d)]
        J = F.jacobian(eta)
        det = np.linalg.det(J)
        if det <= 0:
            raise RuntimeError("geometry error: det J_F <= 0")
        Ji = np.linalg.inv(J)
        C = Ji @ Ji.T
        x = F.value(eta) if (nu_s or gamma_s) else None
        nu = nu_s(x) if nu_s else 1.0
        gam = gamma_s(x) if gamma_s else 1.0
        for l in range(d):
            out[flat + l * n_elems] = C[l, l] * det * nu
        out[flat + d * n_elems] = det * gam
    return out


def separate_variables(samples, nel):
    """assembly.cpp:313-411 (ALS, <= 50 sweeps, tol 1e-10, geometric-mean gauge)."""
    d = len(nel)
    n_elems = int(np.prod(nel))
    samples = np.asarray(samples)
    if (samples <= 0).any():
        raise ValueError("separate_variables: all samples must be positive")
    sl = lambda s: samples[s * n_elems:(s + 1) * n_elems].reshape(nel[::-1]).transpose(range(d)[::-1])  # noqa: E731
    phi = [np.ones(n) for n in nel]
    G = sl(d)  # indexed [i_1, ..., i_d]
    sweeps, converged = 0, False
    for sweep in range(50):
        max_rel = 0.0
        for l in range(d):
            w = np.ones(nel)
            for k in range(d):
                if k != l:
                    shape = [1] * d
                    shape[k] = nel[k]
                    w = w * phi[k].reshape(shape)
            ax = tuple(k for k in range(d) if k != l)
            num = (G * w).sum(axis=ax) if ax else G * w
            den = (w * w).sum(axis=ax) if ax else w * w
            nxt = num / den
            max_rel = max(max_rel, float(np.max(np.abs(nxt - phi[l]) / np.abs(phi[l]))))
            phi[l] = nxt
        sweeps = sweep + 1
        if max_rel <= 1e-10:
            converged = True
            break
    for l in range(1, d):
        g = math.exp(np.log(phi[l]).sum() / nel[l])
        phi[l] = phi[l] / g
        phi[0] = phi[0] * g
    Phi = []
    for l in range(d):
        w = np.ones(nel)
        for k in range(d):
            if k != l:
                shape = [1] * d
                shape[k] = nel[k]
                w = w * phi[k].reshape(shape)
        ax = tuple(k for k in range(d) if k != l)
        E = sl(l)
        acc = (E / w).sum(axis=ax) if ax else E / w
        Phi.append(acc / (n_elems // nel[l]))
    return phi, Phi, sweeps, converged


def assemble_spatial_physical(spaces, F, q, nu_s=None, gamma_s=None):
    """assembly.cpp:151-268 (element loop, pullback with J^-T, triplets summed) -> sparse K, M."""
    d = len(spaces)
    quads = [gauss_rule(s.kv, q) for s in spaces]
    n = [s.dim for s in spaces]
    nel = [qd.num_elements for qd in quads]
    loc = [s.degree + 1 for s in spaces]
    tabs = []
    for s, qd in zip(spaces, quads):
        first, val, der = [], [], []
        for x in qd.nodes:
            f, v = s.eval_active(x, 0)
            _, dv = s.eval_active(x, 1)
            first.append(f)
            val.append(v)
            der.append(dv)
        tabs.append((first, np.array(val), np.array(der)))
    strides = [int(np.prod(n[:l])) for l in range(d)]
    N = int(np.prod(n))
    rows, cols, kv_, mv_ = [], [], [], []
    for e in _multi(nel):
        gidx = []
        for a in _multi(loc):
            g, ok = 0, True
            for l in range(d):
                act = tabs[l][0][e[l] * q] + a[l]
                if act < 0 or act >= n[l]:
                    ok = False
                    break
                g += act * strides[l]
            gidx.append(g if ok else -1)
        L = len(gidx)
        Kl, Ml = np.zeros((L, L)), np.zeros((L, L))
        for j in _multi([q] * d):
            qp = [e[l] * q + j[l] for l in range(d)]
            eta = [quads[l].nodes[qp[l]] for l in range(d)]
            w = float(np.prod([quads[l].weights[qp[l]] for l in range(d)]))
            J = F.jacobian(eta)
            det = np.linalg.det(J)
            JinvT = np.linalg.inv(J).T
            x = F.value(eta) if (nu_s or gamma_s) else None
            nu = nu_s(x) if nu_s else 1.0
            gam = gamma_s(x) if gamma_s else 1.0
            Bv = np.zeros(L)
            Bg = np.zeros((d, L))
            for li, a in enumerate(_multi(loc)):
                Bv[li] = np.prod([tabs[l][1][qp[l], a[l]] for l in range(d)])
                for c in range(d):
                    Bg[c, li] = np.prod([tabs[l][2][qp[l], a[l]] if l == c else tabs[l][1][qp[l], a[l]]
                                         for l in range(d)])
            G = JinvT @ Bg
            Kl += w * det * nu * (G.T @ G)
            Ml += w * det * gam * np.outer(Bv, Bv)
        for a in range(L):
            if gidx[a] < 0:
                continue
            for b in range(L):
                if gidx[b] < 0:
                    continue
                rows.append(gidx[a])
                cols.append(gidx[b])
                kv_.append(Kl[a, b])
                mv_.append(Ml[a, b])
    K = sp.csr_matrix((kv_, (rows, cols)), shape=(N, N))
    M = sp.csr_matrix((mv_, (rows, cols)), shape=(N, N))
    return K, M


def geometry_preconditioner_pieces(prob, p, n_el, want_system=True):
    """SpaceTimeSystem (solver.cpp:34-120) + make_geometry_preconditioner (solver.cpp:127-144):
    returns dict(Kt, Mt_s, Wt, Mt, D, phi, Phi, Ks, Ms)."""
    d, q, T = prob.d, p + 1, prob.T
    spaces = [SplineSpace1D.spatial(p, n_el) for _ in range(d)]
    kvs = [s.kv for s in spaces]
    Wt, Mplain = assemble_time_matrices(p, n_el, T)
    if prob.nu_t or prob.gamma_t:
        ts = SplineSpace1D.temporal(p, n_el)
        tw = lambda tau: (prob.nu_t(T * tau) if prob.nu_t else 1.0) / (prob.gamma_t(T * tau) if prob.gamma_t else 1.0)  # noqa: E731
        Mt = T * assemble_univariate(ts, gauss_rule(ts.kv, q), 0, 0, weight_at=tw)
    else:
        Mt = Mplain
    phi, Phi, _, _ = separate_variables(coefficient_diagonal_samples(kvs, prob.geometry, prob.nu_s, prob.gamma_s),
                                        [n_el] * d)
    Kt = [assemble_univariate(spaces[l], gauss_rule(kvs[l], q), 1, 1, element_weights=Phi[l]) for l in range(d)]
    Mts = [assemble_univariate(spaces[l], gauss_rule(kvs[l], q), 0, 0, element_weights=phi[l]) for l in range(d)]
    out = dict(Kt=Kt, Mt_s=Mts, Wt=Wt, Mt=Mt, phi=phi, Phi=Phi)
    if want_system:
        Ks, Ms = assemble_spatial_physical(spaces, prob.geometry, q, prob.nu_s, prob.gamma_s)
        diagA = np.kron(np.diag(Wt), Ms.diagonal()) + np.kron(np.diag(Mt), Ks.diagonal())
        diagAt = np.zeros_like(diagA)
        for c, fs in kron_sum_terms(Kt, Mts, Wt, Mt, 1.0, 1.0):
            acc = np.ones(1)
            for f in fs:
                acc = np.kron(np.diag(f), acc)
            diagAt += c * acc
        out.update(D=diagA / diagAt, Ks=Ks, Ms=Ms)
    return out
