"""SpaceTimeSystem glue around the hot path (solver.cpp:34-155): A-hat's quadrature means, the RHS
(assemble_rhs, assembly.cpp:413-504) and the error norms (compute_errors, problems.cpp:305-402).

CPU: the oracle restatement is pinned by the convergence orders of the manufactured problems
(L2(L2) ~ h^(p+1), X-norm ~ h^p) and the host means against the oracle.  GPU: the device RHS and error
kernels against the oracle, and the whole SpaceTimeSystem solve (A-hat and A-hat-G) against the oracle's
iteration counts and errors."""
import math

import numpy as np
import pytest

from oracle import problems as opr
from paper_1909_07309_b200 import _lib
from paper_1909_07309_b200 import problems as pp

CATALOG = ["identity-interval-1d", "identity-square-2d", "quarter-annulus-2d", "separable-nu-2d", "deformed-cube-3d"]


@pytest.mark.parametrize("pid", CATALOG)
@pytest.mark.parametrize("p,n_el", [(2, 3), (3, 4)])
def test_system_means_match_oracle(pid, p, n_el):
    prob = opr.make_full_problem(pid)
    g, n = opr.system_means(prob, p, n_el)
    gd, nd = pp.system_means(pid, p, n_el)
    assert abs(gd - g) <= 1e-14 * abs(g) and abs(nd - n) <= 1e-13 * abs(n)
    if pid == "separable-nu-2d":
        assert n > 100.0  # nu_t ~ 101 dominates: A-hat's nu_bar != 1 exercises the c1*c1/nu quirk


def test_problem_info():
    assert pp.problem_info("quarter-annulus-2d")[:4] == (2, 1.0, True, True)
    assert pp.problem_info("deformed-cube-3d")[:4] == (3, 1.0, False, False)


def test_rhs_and_errors_without_source_are_invalid_argument():
    import ctypes

    prob = pp.Problem("deformed-cube-3d")
    st = _lib.lib().stiga_assemble_rhs(prob._h, 2, 2, 3, 0, ctypes.c_void_p(8), None)
    assert st == _lib.INVALID_ARGUMENT
    st = _lib.lib().stiga_compute_errors(prob._h, 2, 2, ctypes.c_void_p(8), 5, 0, ctypes.pointer(ctypes.c_double()),
                                         ctypes.pointer(ctypes.c_double()))
    assert st == _lib.INVALID_ARGUMENT


@pytest.mark.parametrize("pid", ["identity-square-2d", "quarter-annulus-2d"])
def test_oracle_convergence_orders(pid):
    """Known answer of the Galerkin method (PAPER.md a-priori estimates): with p = 2, halving h divides
    the L2(L2) error by ~2^(p+1) and the X-norm bound by ~2^p."""
    prob = opr.make_full_problem(pid)
    errs = []
    for n_el in (4, 8):
        sysm = opr.SpaceTimeSystem(prob, 2, n_el)
        x, rep = sysm.solve(sysm.make_geometry_preconditioner(), tol=1e-12, max_krylov=200)
        assert rep.converged
        errs.append(opr.compute_errors(x, sysm.spaces, sysm.tspace, prob, 5))
    o_l2 = math.log2(errs[0][0] / errs[1][0])
    o_x = math.log2(errs[0][1] / errs[1][1])
    assert 2.8 < o_l2 < 3.6, o_l2
    assert 1.8 < o_x < 2.5, o_x


# ---- device ----------------------------------------------------------------------------------------
RHS_CASES = [("identity-interval-1d", 3, 6, None), ("identity-square-2d", 2, 4, None),
             ("identity-square-2d", 3, 3, 6), ("quarter-annulus-2d", 2, 4, None), ("separable-nu-2d", 2, 3, None),
             ("identity-cube-3d", 2, 2, None)]


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,n_el,ppe", RHS_CASES)
def test_device_rhs_matches_oracle(pid, p, n_el, ppe):
    prob = opr.make_full_problem(pid)
    from oracle.bspline import SplineSpace1D

    spaces = [SplineSpace1D.spatial(p, n_el) for _ in range(prob.d)]
    ts = SplineSpace1D.temporal(p, n_el)
    bo = opr.assemble_rhs(prob.rhs, prob.T, spaces, ts, prob.geometry, ppe or p + 1)
    bd = pp.assemble_rhs(pid, p, n_el, points_per_element=ppe).cpu().numpy()
    rel = np.linalg.norm(bd - bo) / np.linalg.norm(bo)
    assert rel <= 1e-12, rel


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,n_el", [("identity-interval-1d", 2, 4), ("identity-square-2d", 2, 4),
                                        ("quarter-annulus-2d", 2, 3), ("separable-nu-2d", 3, 3),
                                        ("identity-cube-3d", 2, 2)])
def test_device_errors_match_oracle(pid, p, n_el):
    import torch

    prob = opr.make_full_problem(pid)
    sysm = opr.SpaceTimeSystem(prob, p, n_el)
    x, rep = sysm.solve(sysm.make_geometry_preconditioner(), tol=1e-12, max_krylov=300)
    eo = opr.compute_errors(x, sysm.spaces, sysm.tspace, prob, p + 3)
    uh = pp.DiscreteSolution(torch.from_numpy(x).cuda(), pp.Problem(pid), p, n_el)
    ed = pp.compute_errors(uh)
    for a, b in zip(ed, eo):
        assert abs(a - b) <= 1e-11 * b, (ed, eo)
    # a coarser / richer rule (batching over time points differs)
    ed2 = pp.compute_errors(uh, points_per_element=p + 1)
    eo2 = opr.compute_errors(x, sysm.spaces, sysm.tspace, prob, p + 1)
    for a, b in zip(ed2, eo2):
        assert abs(a - b) <= 1e-11 * b, (ed2, eo2)


@pytest.mark.gpu
@pytest.mark.parametrize("pid", ["quarter-annulus-2d", "separable-nu-2d", "identity-square-2d"])
@pytest.mark.parametrize("which", ["parametric", "geometry"])
def test_spacetime_system_solve_matches_oracle(pid, which):
    """SpaceTimeSystem::solve (solver.cpp:146-155) with A-hat (make_parametric_preconditioner: mean
    coefficients, nu_bar >> 1 on separable-nu) or A-hat-G: iteration count +-1 and the error norms."""
    from paper_1909_07309_b200 import stiga

    p, n_el = 2, 8
    prob = opr.make_full_problem(pid)
    so = opr.SpaceTimeSystem(prob, p, n_el)
    Po = so.make_parametric_preconditioner() if which == "parametric" else so.make_geometry_preconditioner()
    xo, ro = so.solve(Po, tol=1e-8, max_krylov=300, restart=50)
    eo = opr.compute_errors(xo, so.spaces, so.tspace, prob, p + 3)

    sd = pp.SpaceTimeSystem(pid, p, n_el, device=0)
    assert abs(sd.gamma_mean - so.gamma_mean) <= 1e-14 and abs(sd.nu_mean - so.nu_mean) <= 1e-12 * so.nu_mean
    bo = so.b
    bd = sd.rhs().cpu().numpy()
    assert np.linalg.norm(bd - bo) <= 1e-12 * np.linalg.norm(bo)
    Pd = sd.make_parametric_preconditioner() if which == "parametric" else sd.make_geometry_preconditioner()
    uh, rd = sd.solve(Pd, stiga.GmresOptions(tol=1e-8, max_krylov=300, restart=50))
    assert rd.converged and abs(rd.iterations - ro.iterations) <= 1, (rd.iterations, ro.iterations)
    ed = pp.compute_errors(uh)
    for a, b in zip(ed, eo):
        assert abs(a - b) <= 1e-6 * b, (ed, eo)  # two GMRES runs to 1e-8: errors agree to the solve tolerance


@pytest.mark.gpu
def test_device_convergence_orders_3d():
    """identity-cube-3d end to end on the device (RHS, A-hat-G solve, errors): orders p+1 and p."""
    from paper_1909_07309_b200 import stiga

    p, errs = 2, []
    for n_el in (4, 8, 16):
        sd = pp.SpaceTimeSystem("identity-cube-3d", p, n_el)
        uh, rep = sd.solve(sd.make_geometry_preconditioner(), stiga.GmresOptions(tol=1e-12, max_krylov=50))
        assert rep.converged
        errs.append(pp.compute_errors(uh))
    o_l2 = math.log2(errs[1][0] / errs[2][0])
    o_x = math.log2(errs[1][1] / errs[2][1])
    assert 2.7 < o_l2 < 3.5 and 1.8 < o_x < 2.4, (errs, o_l2, o_x)
