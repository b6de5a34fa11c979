"""Space-time system glue, right-hand side and error norms (oracle, test infrastructure only).

Follows /root/reference/proj/core/src:
  problems.cpp:126-241   exact solutions / source terms of the catalog (identity_problem,
                         quarter_annulus_problem, separable_nu_problem)
  assembly.cpp:413-504   assemble_rhs (element loop, Gauss rule, f(x, T tau) pulled back)
  solver.cpp:34-125      SpaceTimeSystem: A_, b_, the quadrature means gamma_mean / nu_mean,
                         make_parametric_preconditioner / make_geometry_preconditioner
  solver.cpp:146-155     SpaceTimeSystem::solve (left-preconditioned GMRES from x0 = 0)
  problems.cpp:263-402   DiscreteSolution::eval_parametric, compute_errors
The deformed cube of BASELINE config 4 carries no manufactured solution (its RHS is seeded).
"""
import math

import numpy as np
import scipy.sparse as sp

from .assembly import assemble_spatial_parametric, assemble_time_matrices, assemble_univariate
from .bspline import SplineSpace1D, gauss_rule
from .fdsolve import ExtendedFDPreconditioner
from .geometry import _multi, assemble_spatial_physical, geometry_preconditioner_pieces, make_problem
from .gmres import gmres
from .kronop import mode_product

PI = math.pi


# ---- manufactured solutions (problems.cpp:131-241) ---------------------------------------------
def _identity_exact(d):
    def spatial(x):
        v = 1.0
        for l in range(d):
            v *= math.sin(PI * x[l])
        return v

    def u(x, t):
        return spatial(x) * math.sin(PI * t)

    def du_dt(x, t):
        return spatial(x) * PI * math.cos(PI * t)

    def grad_u(x, t):
        g = np.zeros(d)
        for l in range(d):
            v = PI * math.cos(PI * x[l])
            for k in range(d):
                if k != l:
                    v *= math.sin(PI * x[k])
            g[l] = v * math.sin(PI * t)
        return g

    def rhs(x, t):
        return spatial(x) * (PI * math.cos(PI * t) + d * PI * PI * math.sin(PI * t))

    return rhs, (u, grad_u, du_dt)


def _annulus_P(x1, x2):
    r2 = x1 * x1 + x2 * x2
    return -(r2 - 1.0) * (r2 - 4.0) * x1 * x2 * x2


def _annulus_dP(x1, x2):
    a, b = x1 * x1, x2 * x2
    d1 = -5.0 * a * a * b - 6.0 * a * b * b + 15.0 * a * b - b * b * b + 5.0 * b * b - 4.0 * b
    d2 = (-2.0 * x1 ** 5 * x2 - 8.0 * x1 ** 3 * x2 ** 3 + 10.0 * x1 ** 3 * x2 - 6.0 * x1 * x2 ** 5
          + 20.0 * x1 * x2 ** 3 - 8.0 * x1 * x2)
    return d1, d2


def _annulus_lap(x1, x2):
    return (-2.0 * x1 ** 5 - 44.0 * x1 ** 3 * x2 * x2 + 10.0 * x1 ** 3 - 42.0 * x1 * x2 ** 4
            + 90.0 * x1 * x2 * x2 - 8.0 * x1)


def _annulus_exact():
    def u(x, t):
        return _annulus_P(x[0], x[1]) * math.sin(t)

    def du_dt(x, t):
        return _annulus_P(x[0], x[1]) * math.cos(t)

    def grad_u(x, t):
        return np.array(_annulus_dP(x[0], x[1])) * math.sin(t)

    def rhs(x, t):
        return _annulus_P(x[0], x[1]) * math.cos(t) - _annulus_lap(x[0], x[1]) * math.sin(t)

    return rhs, (u, grad_u, du_dt)


def _separable_nu_rhs(nu_s, nu_t):
    def rhs(x, t):
        s1, c1 = math.sin(PI * x[0]), math.cos(PI * x[0])
        s2, c2 = math.sin(PI * x[1]), math.cos(PI * x[1])
        st, ct = math.sin(PI * t), math.cos(PI * t)
        r = math.hypot(x[0], x[1])
        r3 = r * r * r
        dnu1 = -49.5 * x[0] * x[1] / r3
        dnu2 = 49.5 * x[0] * x[0] / r3
        lap_u = -2.0 * PI * PI * s1 * s2 * st
        gdot = dnu1 * PI * c1 * s2 * st + dnu2 * PI * s1 * c2 * st
        return PI * s1 * s2 * ct - nu_t(t) * (nu_s(x) * lap_u + gdot)

    return rhs


def make_full_problem(pid):
    """make_problem(id) (problems.cpp:244-261) with the source term and exact solution attached
    (prob.rhs, prob.exact = (u, grad_u, du_dt) or None) and gamma0 = nu0 = 1."""
    prob = make_problem(pid)
    prob.gamma0 = prob.nu0 = 1.0
    prob.rhs, prob.exact = None, None
    if pid.startswith("identity-"):
        prob.rhs, prob.exact = _identity_exact(prob.d)
    elif pid == "quarter-annulus-2d":
        prob.rhs, prob.exact = _annulus_exact()
    elif pid == "separable-nu-2d":
        _, prob.exact = _identity_exact(2)
        prob.rhs = _separable_nu_rhs(prob.nu_s, prob.nu_t)
    return prob


# ---- assemble_rhs (assembly.cpp:413-504) --------------------------------------------------------
def _tabulate(space, quad):
    first, val, der = [], [], []
    for x in quad.nodes:
        f, v = space.eval_active(x, 0)
        _, dv = space.eval_active(x, 1)
        first.append(f)
        val.append(v)
        der.append(dv)
    return np.array(first), np.array(val), np.array(der)


def assemble_rhs(f, T, spaces, tspace, geometry, ppe):
    """b_(i, it) = sum_e sum_qp w det T w_t f(F(eta), T tau) B_i(eta) b_it(tau), in the reference's
    element / quadrature-point / time-point / local-function loop order."""
    d = len(spaces)
    quads = [gauss_rule(s.kv, ppe) for s in spaces]
    tabs = [_tabulate(s, qd) for s, qd in zip(spaces, quads)]
    n = [s.dim for s in spaces]
    nel = [qd.num_elements for qd in quads]
    loc = [s.degree + 1 for s in spaces]
    tq = gauss_rule(tspace.kv, ppe)
    tfirst, tval, _ = _tabulate(tspace, tq)
    n_t, pt = tspace.dim, tspace.degree
    strides = [int(np.prod(n[:l])) for l in range(d)]
    n_s = int(np.prod(n))
    b = np.zeros(n_s * n_t)
    q = ppe
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
        gidx = np.array(gidx)
        live = gidx >= 0
        for j in _multi([q] * d):
            qp = [e[l] * q + j[l] for l in range(d)]
            eta = [quads[l].nodes[qp[l]] for l in range(d)]
            w = 1.0
            for l in range(d):
                w *= quads[l].weights[qp[l]]
            det = np.linalg.det(geometry.jacobian(eta))
            if det <= 0.0:
                raise RuntimeError("assemble_rhs: non-positive Jacobian determinant")
            x = geometry.value(eta)
            Bval = np.array([np.prod([tabs[l][1][qp[l], a[l]] for l in range(d)]) for a in _multi(loc)])
            wx = w * det * T
            for qt in range(tq.num_points):
                c = wx * tq.weights[qt] * f(x, T * tq.nodes[qt])
                for at in range(pt + 1):
                    it = tfirst[qt] + at
                    if it < 0 or it >= n_t:
                        continue
                    ct = c * tval[qt, at]
                    if ct == 0.0:
                        continue
                    np.add.at(b, gidx[live] + it * n_s, ct * Bval[live])
    return b


# ---- SpaceTimeSystem (solver.cpp:34-155) ---------------------------------------------------------
def system_means(prob, p, n_el):
    """gamma_mean = int gamma_s / |Omega|, nu_mean = int nu_s / |Omega| * int_0^1 nu_t/gamma_t
    (solver.cpp:82-112, Gauss rule with q = p + 1 points, tensor loop direction 0 fastest)."""
    d, q, T = prob.d, p + 1, prob.T
    rules = [gauss_rule(SplineSpace1D.spatial(p, n_el).kv, q) for _ in range(d)]
    vol = g_int = n_int = 0.0
    for idx in _multi([r.num_points for r in rules]):
        eta = [rules[l].nodes[idx[l]] for l in range(d)]
        w = 1.0
        for l in range(d):
            w *= rules[l].weights[idx[l]]
        det = np.linalg.det(prob.geometry.jacobian(eta))
        x = prob.geometry.value(eta)
        vol += w * det
        g_int += w * det * (prob.gamma_s(x) if prob.gamma_s else 1.0)
        n_int += w * det * (prob.nu_s(x) if prob.nu_s else 1.0)
    tq = gauss_rule(SplineSpace1D.temporal(p, n_el).kv, q)
    t_mean = 0.0
    for qt in range(tq.num_points):
        tau = tq.nodes[qt]
        nt = prob.nu_t(T * tau) if prob.nu_t else 1.0
        gt = prob.gamma_t(T * tau) if prob.gamma_t else 1.0
        t_mean += tq.weights[qt] * nt / gt
    return g_int / vol, n_int / vol * t_mean


class SpaceTimeSystem:
    """solver.hpp:13-58 on the CPU (small sizes): physical A_, analytic b_, both preconditioners."""

    def __init__(self, prob, p, n_el):
        self.prob, self.p, self.n_el = prob, p, n_el
        d, T = prob.d, prob.T
        self.spaces = [SplineSpace1D.spatial(p, n_el) for _ in range(d)]
        self.tspace = SplineSpace1D.temporal(p, n_el)
        pcs = geometry_preconditioner_pieces(prob, p, n_el, want_system=True)
        self.pieces = pcs
        self.Wt, self.Mt = pcs["Wt"], pcs["Mt"]
        _, self.Mt_plain = assemble_time_matrices(p, n_el, T)
        self.Ks, self.Ms = pcs["Ks"], pcs["Ms"]
        self.A = (sp.kron(sp.csr_matrix(self.Wt), self.Ms) + sp.kron(sp.csr_matrix(self.Mt), self.Ks)).tocsr()
        f = prob.rhs
        gt = prob.gamma_t
        rhs = f if gt is None else (lambda x, t: f(x, t) / gt(t))
        self.b = assemble_rhs(rhs, T, self.spaces, self.tspace, prob.geometry, p + 1) if f else None
        self.gamma_mean, self.nu_mean = system_means(prob, p, n_el)

    @property
    def n_dof(self):
        return self.A.shape[0]

    def make_parametric_preconditioner(self):
        """solver.cpp:122-125: setup(K^, M^, W_t, plain M_t, gamma_mean, nu_mean)."""
        K, M = assemble_spatial_parametric(self.p, self.n_el, self.prob.d, q=self.p + 1)
        return ExtendedFDPreconditioner.setup(K, M, self.Wt, self.Mt_plain, self.gamma_mean, self.nu_mean)

    def make_geometry_preconditioner(self):
        """solver.cpp:127-144."""
        pc = self.pieces
        return ExtendedFDPreconditioner.setup(pc["Kt"], pc["Mt_s"], pc["Wt"], pc["Mt"], 1.0, 1.0, scaling=pc["D"])

    def solve(self, P, tol=1e-8, max_krylov=100, restart=None):
        """solver.cpp:146-155."""
        x, rep = gmres(lambda v: self.A @ v, (lambda v: P.apply(v)) if P is not None else None, self.b,
                       tol=tol, max_krylov=max_krylov, restart=restart)
        return x, rep


# ---- compute_errors (problems.cpp:305-402) -------------------------------------------------------
def collocation_active(space, pts, deriv):
    """problems.cpp:35-49."""
    B = np.zeros((len(pts), space.dim))
    for qi, x in enumerate(pts):
        first, v = space.eval_active(x, deriv)
        for r in range(space.degree + 1):
            j = first + r
            if 0 <= j < space.dim:
                B[qi, j] = v[r]
    return B


def eval_parametric(coeffs, spaces, tspace, eta, tau):
    """DiscreteSolution::eval_parametric (problems.cpp:263-303)."""
    d = len(spaces)
    n = [s.dim for s in spaces]
    n_s = int(np.prod(n))
    tf, tv = tspace.eval_active(tau, 0)
    tot = 0.0
    evs = [s.eval_active(eta[l], 0) for l, s in enumerate(spaces)]
    for at in range(tspace.degree + 1):
        it = tf + at
        if it < 0 or it >= tspace.dim or tv[at] == 0.0:
            continue
        for a in _multi([s.degree + 1 for s in spaces]):
            v, g, ok = tv[at], it * n_s, True
            stride = 1
            for l in range(d):
                act = evs[l][0] + a[l]
                if act < 0 or act >= n[l]:
                    ok = False
                    break
                v *= evs[l][1][a[l]]
                g += act * stride
                stride *= n[l]
            if ok:
                tot += v * coeffs[g]
    return tot


def compute_errors(coeffs, spaces, tspace, prob, ppe):
    """Relative L2(0,T;L2) error and X-norm upper bound (problems.cpp:305-402)."""
    if prob.exact is None:
        raise ValueError("compute_errors: problem has no exact solution")
    d, T = len(spaces), prob.T
    gamma, nu = prob.gamma0, prob.nu0
    wt_dt = gamma * gamma / nu
    quads = [gauss_rule(s.kv, ppe) for s in spaces]
    tq = gauss_rule(tspace.kv, ppe)
    dims = [s.dim for s in spaces] + [tspace.dim]
    val_ops = [collocation_active(s, qd.nodes, 0) for s, qd in zip(spaces, quads)] + \
              [collocation_active(tspace, tq.nodes, 0)]
    der_ops = [collocation_active(s, qd.nodes, 1) for s, qd in zip(spaces, quads)] + \
              [collocation_active(tspace, tq.nodes, 1)]

    def grid(slot):
        x, dd = np.asarray(coeffs, dtype=np.float64), list(dims)
        for m in range(d + 1):
            J = der_ops[m] if slot == m else val_ops[m]
            x, dd = mode_product(x, dd, J, m)
        return x

    V = grid(-1)
    G = [grid(l) for l in range(d)]
    Vt = grid(d)
    npts = [qd.num_points for qd in quads]
    n_sp = int(np.prod(npts))
    xs, JinvT, dets, wsp = [], [], np.zeros(n_sp), np.zeros(n_sp)
    for flat, idx in enumerate(_multi(npts)):
        eta = [quads[l].nodes[idx[l]] for l in range(d)]
        w = 1.0
        for l in range(d):
            w *= quads[l].weights[idx[l]]
        J = prob.geometry.jacobian(eta)
        dets[flat] = np.linalg.det(J)
        if dets[flat] <= 0.0:
            raise RuntimeError("compute_errors: non-positive Jacobian determinant")
        JinvT.append(np.linalg.inv(J).T)
        xs.append(prob.geometry.value(eta))
        wsp[flat] = w
    u, grad_u, du_dt = prob.exact
    l2n = l2d = xn = xd = 0.0
    for qt in range(tq.num_points):
        t = T * tq.nodes[qt]
        wt = tq.weights[qt] * T
        off = qt * n_sp
        for js in range(n_sp):
            w = wt * wsp[js] * dets[js]
            ue, dte, ge = u(xs[js], t), du_dt(xs[js], t), grad_u(xs[js], t)
            e = V[off + js] - ue
            de = Vt[off + js] / T - dte
            gh = np.array([G[l][off + js] for l in range(d)])
            gerr = JinvT[js] @ gh - ge
            l2n += w * e * e
            l2d += w * ue * ue
            xn += w * (wt_dt * de * de + nu * float(gerr @ gerr))
            xd += w * (wt_dt * dte * dte + nu * float(ge @ ge))
    if l2d == 0.0 or xd == 0.0:
        raise ValueError("compute_errors: exact solution has zero norm")
    return math.sqrt(l2n / l2d), math.sqrt(xn / xd)
