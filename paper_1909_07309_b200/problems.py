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


def kron_sum_diagonal(terms, t_range=None):
    """KronSumOperator::diagonal (kronop.cpp:117-131): sum_t c_t kron(diag F_D, ..., diag F_1).
    t_range = (t0, t1): only the slices t0 <= t < t1 of the last (slowest) mode -- a rank's time slab."""
    out = None
    for c, fs in terms:
        acc = np.ones(1)
        for k, f in enumerate(fs):
            dg = np.diag(f)
            if t_range is not None and k == len(fs) - 1:
                dg = dg[t_range[0]:t_range[1]]
            acc = np.kron(dg, acc)
        out = c * acc if out is None else out + c * acc
    return out


def geometry_scaling(pc, K_tilde=None, M_tilde=None, Mt_tilde=None, t_range=None):
    """D = diag(A) / diag(A~) with A~ in (d+1)-factor form (solver.cpp:138-142).  On the identity
    map with constant coefficients K~ = K, M~ = M and D == 1.  t_range: a time slab of it."""
    A = stiga.kron_sum_terms(pc.K, pc.M, pc.Wt, pc.Mt, pc.gamma, pc.nu)
    At = stiga.kron_sum_terms(K_tilde or pc.K, M_tilde or pc.M, pc.Wt,
                              pc.Mt if Mt_tilde is None else Mt_tilde, 1.0, 1.0)
    return kron_sum_diagonal(A, t_range) / kron_sum_diagonal(At, t_range)


class Problem:
    """make_problem(id) (problems.cpp:244-261) on the host through the C ABI; the geometry map and
    coefficient fields are native (they are evaluated at every quadrature point of the setup)."""

    def __init__(self, pid):
        import ctypes

        from ._lib import check, lib

        self._lib, self._check, self._ct = lib, check, ctypes
        h = ctypes.c_void_p()
        check(lib().stiga_problem_create(pid.encode(), ctypes.byref(h)), "make_problem")
        self._h = h
        d = ctypes.c_int()
        check(lib().stiga_problem_dim(h, ctypes.byref(d)), "problem_dim")
        self.d = d.value
        self.name = pid

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib().stiga_problem_destroy(h)
            except Exception:
                pass
            self._h = None

    def _p(self, a):
        return a.ctypes.data_as(self._ct.POINTER(self._ct.c_double))

    def geometry(self, eta):
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        x = np.zeros(self.d)
        J = np.zeros(self.d * self.d)
        self._check(self._lib().stiga_problem_eval_geometry(self._h, self._p(eta), self._p(x), self._p(J)), "geometry")
        return x, J.reshape(self.d, self.d).T.copy()

    def fields(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        nu, gam = self._ct.c_double(), self._ct.c_double()
        self._check(self._lib().stiga_problem_eval_fields(self._h, self._p(x), self._ct.byref(nu), self._ct.byref(gam)),
                    "fields")
        return nu.value, gam.value

    def geometry_pieces(self, p, n_el, want_D=True, device=None, D_on_device=False):
        """make_geometry_preconditioner inputs (solver.cpp:127-144): SpaceTimePieces with the
        separated-coefficient factors K~, M~, W_t, weighted M_t, plus D and phi/Phi.

        device=None: D = diag(A)/diag(A~) with diag(A) from the host quadrature of the physical
        diagonal.  device=k: diag(A) from the physical K_s, M_s assembled on GPU k (the operator the
        GMRES solve applies; `pc.A` keeps it) -- the same quadrature sums in another order, seconds
        instead of the host's per-element loop at c4 sizes.  The ratio itself is formed on the device
        (stiga_geometry_scaling_device, bit-identical to the host division); D_on_device=True keeps D
        there as a CUDA tensor (ExtendedFDPreconditioner.setup then forms D^-1/2 on the device)."""
        if want_D and device is not None:
            pc = self.geometry_pieces(p, n_el, want_D=False)
            A = stiga.KronSumOperator.physical(self, p, n_el, device=device)
            At = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=device)
            Dd = stiga.geometry_scaling_device(A, At)
            pc.D = Dd if D_on_device else Dd.cpu().numpy()
            pc.A = A
            return pc
        ns = stiga.space_dim(p, n_el)
        nt = stiga.space_dim(p, n_el, temporal=True)
        d = self.d
        Kt = np.zeros(d * ns * ns)
        Ms = np.zeros(d * ns * ns)
        Wt = np.zeros(nt * nt)
        Mt = np.zeros(nt * nt)
        D = np.zeros(ns ** d * nt) if want_D else None
        phi = np.zeros(d * n_el)
        Phi = np.zeros(d * n_el)
        res = np.zeros(d + 1)
        sweeps = self._ct.c_int()
        self._check(self._lib().stiga_geometry_preconditioner_pieces(
            self._h, p, n_el, self._p(Kt), self._p(Ms), self._p(Wt), self._p(Mt),
            self._p(D) if D is not None else None, self._p(phi), self._p(Phi), self._p(res),
            self._ct.byref(sweeps)), "geometry_preconditioner_pieces")
        blk = lambda a, l: a[l * ns * ns:(l + 1) * ns * ns].reshape(ns, ns).T.copy()  # noqa: E731
        pc = SpaceTimePieces(d, p, n_el, [blk(Kt, l) for l in range(d)], [blk(Ms, l) for l in range(d)],
                             Wt.reshape(nt, nt).T.copy(), Mt.reshape(nt, nt).T.copy())
        pc.D = D
        pc.phi = phi.reshape(d, n_el)
        pc.Phi = Phi.reshape(d, n_el)
        pc.residuals = res
        pc.sweeps = sweeps.value
        return pc


# ------------------------------------------------------------------------------------------------
# SpaceTimeSystem (solver.hpp:13-58) on the device
# ------------------------------------------------------------------------------------------------
def _as_problem(problem):
    return Problem(problem) if isinstance(problem, str) else problem


def problem_info(problem):
    """(d, T, has_rhs, has_exact, gamma0, nu0) of a catalog problem (problems.hpp:25-37)."""
    import ctypes

    from ._lib import check, lib

    problem = _as_problem(problem)
    d, hr, he = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    T, g0, n0 = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().stiga_problem_info(problem._h, ctypes.byref(d), ctypes.byref(T), ctypes.byref(hr), ctypes.byref(he),
                                   ctypes.byref(g0), ctypes.byref(n0)), "problem_info")
    return d.value, T.value, bool(hr.value), bool(he.value), g0.value, n0.value


def system_means(problem, p, n_el):
    """SpaceTimeSystem::gamma_mean() / nu_mean() (solver.cpp:82-112)."""
    import ctypes

    from ._lib import check, lib

    problem = _as_problem(problem)
    g, n = ctypes.c_double(), ctypes.c_double()
    check(lib().stiga_system_means(problem._h, int(p), int(n_el), ctypes.byref(g), ctypes.byref(n)), "system_means")
    return g.value, n.value


def assemble_rhs(problem, p, n_el, points_per_element=None, device=0, out=None):
    """b_ of SpaceTimeSystem (solver.cpp:72-76 -> assemble_rhs, assembly.cpp:413-504), sum-factorized
    on the device; returns a float64 CUDA tensor of N_dof (colex, time slowest)."""
    import ctypes

    import torch

    from ._lib import check, lib

    problem = _as_problem(problem)
    ns = stiga.space_dim(p, n_el) ** problem.d
    nt = stiga.space_dim(p, n_el, temporal=True)
    if out is None:
        out = torch.empty(ns * nt, dtype=torch.float64, device=f"cuda:{device}")
    if out.numel() != ns * nt:
        raise ValueError("assemble_rhs: output length mismatch")
    ppe = p + 1 if points_per_element is None else int(points_per_element)
    check(lib().stiga_assemble_rhs(problem._h, int(p), int(n_el), ppe, int(device), ctypes.c_void_p(out.data_ptr()),
                                   None), "assemble_rhs")
    return out


class DiscreteSolution:
    """problems.hpp:67-77: Galerkin coefficients (device tensor) + the discretisation they live on."""

    def __init__(self, coefficients, problem, p, n_el):
        self.coefficients, self.problem, self.p, self.n_el = coefficients, problem, p, n_el

    @property
    def n_dof(self):
        return self.coefficients.numel()


def compute_errors(uh, problem=None, points_per_element=None):
    """compute_errors(u_h, problem, points_per_element) (problems.cpp:305-402) on the device:
    (relative L2(0,T;L2) error, relative X-norm upper bound).  Default rule: p + 3 points per element
    (study.cpp:164)."""
    import ctypes

    from ._lib import check, lib

    problem = _as_problem(problem or uh.problem)
    ppe = uh.p + 3 if points_per_element is None else int(points_per_element)
    c = uh.coefficients.contiguous()
    l2, xu = ctypes.c_double(), ctypes.c_double()
    check(lib().stiga_compute_errors(problem._h, int(uh.p), int(uh.n_el), ctypes.c_void_p(c.data_ptr()), ppe,
                                     int(c.device.index or 0), ctypes.byref(l2), ctypes.byref(xu)), "compute_errors")
    return l2.value, xu.value


class SpaceTimeSystem:
    """SpaceTimeSystem(problem, p, n_el) (solver.hpp:13-58, solver.cpp:34-155) on one device.

    A_ is the physical system M_s (x) W_t + K_s (x) M_t: on the identity map with constant coefficients
    (identity-* problems) the sum-factorized Kronecker-sum form (equal in exact arithmetic), otherwise
    the device-assembled physical operator.  b_ is assembled on the device (assemble_rhs above) when the
    problem carries a source term.  Holds the problem by reference like the reference (solver.hpp:46)."""

    def __init__(self, problem, p, n_el, device=0):
        self.problem = _as_problem(problem)
        self.p, self.n_el, self.device = int(p), int(n_el), int(device)
        d, self.T, has_rhs, _, _, _ = problem_info(self.problem)
        self.d = d
        self.gamma_mean, self.nu_mean = system_means(self.problem, p, n_el)
        self._pc = None
        if self.problem.name.startswith("identity-"):
            pc = identity_pieces(d, p, n_el, self.T)
            self.Wt, self.Mt, self.Mt_plain = pc.Wt, pc.Mt, pc.Mt
            self.A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=device)
        else:
            pc = self.problem.geometry_pieces(p, n_el, want_D=True, device=device, D_on_device=True)
            self._pc = pc
            self.Wt, self.Mt = pc.Wt, pc.Mt
            _, self.Mt_plain = stiga.assemble_time_matrices(p, n_el, self.T)
            self.A = pc.A
        self.b = assemble_rhs(self.problem, p, n_el, device=device) if has_rhs else None

    @property
    def n_dof(self):
        return self.A.n_dof

    @property
    def n_s(self):
        return self.A.n_dof // self.A.dims[-1]

    @property
    def n_t(self):
        return self.A.dims[-1]

    def system_operator(self):
        return self.A

    def rhs(self):
        return self.b

    def make_parametric_preconditioner(self):
        """A-hat (solver.cpp:122-125): parametric factors, plain M_t, mean coefficients, no scaling."""
        K, M = stiga.assemble_spatial_parametric(self.p, self.n_el, self.d, q=self.p + 1)
        return stiga.ExtendedFDPreconditioner.setup(K, M, self.Wt, self.Mt_plain, self.gamma_mean, self.nu_mean,
                                                    device=self.device)

    def make_geometry_preconditioner(self):
        """A-hat-G (solver.cpp:127-144): separated factors, weighted M_t, D = diag(A)/diag(A~)."""
        if self._pc is None:
            self._pc = self.problem.geometry_pieces(self.p, self.n_el, want_D=True, device=self.device,
                                                    D_on_device=True)
        pc = self._pc
        return stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D,
                                                    device=self.device, device_schur=True)

    def solve(self, P=None, opts=None, b=None):
        """solver.cpp:146-155: left-preconditioned GMRES from x0 = 0 -> (DiscreteSolution, SolveReport)."""
        rhs = self.b if b is None else b
        if rhs is None:
            raise ValueError("SpaceTimeSystem::solve: the problem has no source term; pass b")
        x, rep = stiga.gmres(self.A, P, rhs, opts or stiga.GmresOptions())
        return DiscreteSolution(x, self.problem, self.p, self.n_el), rep
