"""Config-4 host pieces: geometry fit, coefficient samples, separation, D = diag(A)/diag(A~) --
product (C++) against the oracle (numpy restatement of geometry.cpp / problems.cpp / assembly.cpp)."""
import math

import numpy as np
import pytest

from oracle import geometry as og
from paper_1909_07309_b200.problems import Problem


@pytest.mark.parametrize("pid", ["identity-square-2d", "quarter-annulus-2d", "deformed-cube-3d"])
def test_geometry_map_matches_oracle(pid):
    P, Po = Problem(pid), og.make_problem(pid)
    rng = np.random.default_rng(3)
    for _ in range(20):
        eta = rng.uniform(0, 1, P.d)
        x, J = P.geometry(eta)
        assert np.abs(x - Po.geometry.value(eta)).max() <= 1e-13
        assert np.abs(J - Po.geometry.jacobian(eta)).max() <= 1e-12


def test_deformed_cube_fit_and_fields():
    P = Problem("deformed-cube-3d")
    rng = np.random.default_rng(5)
    for _ in range(30):
        eta = rng.uniform(0, 1, 3)
        x, J = P.geometry(eta)
        b = 0.1 * math.sin(math.pi * eta[0]) * math.sin(math.pi * eta[1]) * math.sin(math.pi * eta[2])
        assert np.abs(x - (eta + b)).max() <= 2e-4  # spline fit (p_g=3, 8 elements) of the analytic map
        assert np.linalg.det(J) > 0
        nu, gam = P.fields(x)
        assert nu == pytest.approx(1 + 0.5 * math.sin(2 * math.pi * x[0]) * math.cos(2 * math.pi * x[1]))
        assert gam == pytest.approx(1 + 0.25 * x[2])
    with pytest.raises(ValueError):
        Problem("no-such-problem")


@pytest.mark.parametrize("pid,p,nel", [("identity-square-2d", 2, 4), ("quarter-annulus-2d", 2, 5),
                                        ("separable-nu-2d", 3, 4), ("deformed-cube-3d", 2, 3)])
def test_geometry_preconditioner_pieces_match_oracle(pid, p, nel):
    P, Po = Problem(pid), og.make_problem(pid)
    pc = P.geometry_pieces(p, nel)
    ref = og.geometry_preconditioner_pieces(Po, p, nel)
    for l in range(P.d):
        assert np.abs(pc.phi[l] - ref["phi"][l]).max() <= 1e-12 * np.abs(ref["phi"][l]).max()
        assert np.abs(pc.Phi[l] - ref["Phi"][l]).max() <= 1e-12 * np.abs(ref["Phi"][l]).max()
        assert np.abs(pc.K[l] - ref["Kt"][l]).max() <= 1e-12 * np.abs(ref["Kt"][l]).max()
        assert np.abs(pc.M[l] - ref["Mt_s"][l]).max() <= 1e-12 * np.abs(ref["Mt_s"][l]).max()
    assert np.abs(pc.Wt - ref["Wt"]).max() <= 1e-14
    assert np.abs(pc.Mt - ref["Mt"]).max() <= 1e-13 * np.abs(ref["Mt"]).max()
    assert np.abs(pc.D - ref["D"]).max() <= 1e-11 * np.abs(ref["D"]).max()
    if pid.startswith("identity"):
        assert np.abs(pc.D - 1.0).max() <= 1e-12  # A~ == A on the parametric domain
    else:
        assert np.abs(pc.D - 1.0).max() > 1e-3


def test_separation_is_exact_on_separable_samples():
    rng = np.random.default_rng(7)
    nel = [3, 4, 5]
    f = [rng.uniform(0.5, 2.0, n) for n in nel]
    G = np.einsum("i,j,k->ijk", *f)
    slices = [G * rng.uniform(0.5, 2.0) for _ in range(3)] + [G]
    samples = np.concatenate([s.transpose(2, 1, 0).reshape(-1) for s in slices])
    phi, Phi, sweeps, conv = og.separate_variables(samples, nel)
    fit = np.einsum("i,j,k->ijk", *phi)
    assert conv and np.abs(fit - G).max() <= 1e-10 * G.max()
    for l in (1, 2):
        assert abs(np.log(phi[l]).mean()) <= 1e-12  # geometric-mean gauge


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,nel", [("deformed-cube-3d", 2, 4), ("deformed-cube-3d", 4, 3), ("quarter-annulus-2d", 3, 9),
                                        ("separable-nu-2d", 2, 8)])
def test_geometry_preconditioner_apply_gpu(pid, p, nel):
    """A^G on curved geometry / variable coefficients (D != 1): device apply vs the oracle
    built from the oracle's own pieces (<= 1e-11)."""
    torch = pytest.importorskip("torch")
    from oracle.fdsolve import ExtendedFDPreconditioner as OracleFD
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.inputs import uniform_pm1

    pc = Problem(pid).geometry_pieces(p, nel)
    ref = og.geometry_preconditioner_pieces(og.make_problem(pid), p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D, device=0)
    Po = OracleFD.setup(ref["Kt"], ref["Mt_s"], ref["Wt"], ref["Mt"], 1.0, 1.0, scaling=ref["D"])
    r = uniform_pm1(P.n_dof, 17)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    so = Po.apply(r)
    assert np.linalg.norm(s - so) / np.linalg.norm(so) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,nel", [("identity-cube-3d", 2, 3), ("deformed-cube-3d", 2, 3), ("deformed-cube-3d", 3, 2),
                                        ("quarter-annulus-2d", 2, 6), ("separable-nu-2d", 3, 5)])
def test_physical_system_matvec_and_gmres(pid, p, nel):
    """Device-assembled physical A (stencil SpMM) vs the oracle's assemble_spatial_physical
    (assembly.cpp:151-268) and GMRES iteration parity (+-1) with the A^G preconditioner."""
    torch = pytest.importorskip("torch")
    from oracle import gmres as ogm
    from oracle.fdsolve import ExtendedFDPreconditioner as OracleFD
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.inputs import uniform_pm1

    prob = Problem(pid)
    ref = og.geometry_preconditioner_pieces(og.make_problem(pid), p, nel)
    A = stiga.KronSumOperator.physical(prob, p, nel)
    Ad = sp_kron(ref)
    x = uniform_pm1(A.n_dof, 3)
    y = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = Ad @ x
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    assert np.abs(A.diagonal() - Ad.diagonal()).max() <= 1e-12 * np.abs(Ad.diagonal()).max()
    pc = prob.geometry_pieces(p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D, device=0)
    Po = OracleFD.setup(ref["Kt"], ref["Mt_s"], ref["Wt"], ref["Mt"], 1.0, 1.0, scaling=ref["D"])
    b = uniform_pm1(A.n_dof, 4)
    xg, rep = stiga.gmres(A, P, torch.from_numpy(b).cuda(), stiga.GmresOptions(1e-8, 300, 50))
    xo, repo = ogm.gmres(lambda v: Ad @ v, Po.apply, b, 1e-8, 300, 50)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 1
    assert np.linalg.norm(xg.cpu().numpy() - xo) <= 1e-6 * np.linalg.norm(xo)


def sp_kron(ref):
    import scipy.sparse as sp

    return (sp.kron(sp.csr_matrix(ref["Wt"]), ref["Ms"]) + sp.kron(sp.csr_matrix(ref["Mt"]), ref["Ks"])).tocsr()


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,nel", [("identity-interval-1d", 5, 200), ("identity-interval-1d", 1, 150),
                                        ("identity-interval-1d", 2, 90), ("quarter-annulus-2d", 4, 9),
                                        ("separable-nu-2d", 5, 4)])
def test_physical_matvec_tiling_edges(pid, p, nel):
    """Tensor-core stencil mat-vec at sizes that exercise its tiling: several 96-row segments per
    line and several 72-column time chunks (1D, n up to 203), every band width KS = 3..5 (p = 1..5),
    and partial row blocks / time tiles; against the oracle's assembled A (solver.cpp:67-70)."""
    torch = pytest.importorskip("torch")
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.inputs import uniform_pm1

    prob = Problem(pid)
    ref = og.geometry_preconditioner_pieces(og.make_problem(pid), p, nel)
    A = stiga.KronSumOperator.physical(prob, p, nel)
    Ad = sp_kron(ref)
    for seed in (5, 6):
        x = uniform_pm1(A.n_dof, seed)
        y = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        yo = Ad @ x
        assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)


@pytest.mark.gpu
@pytest.mark.parametrize("pid,p,nel", [("deformed-cube-3d", 2, 4), ("deformed-cube-3d", 4, 6), ("deformed-cube-3d", 3, 5),
                                        ("deformed-cube-3d", 5, 5), ("deformed-cube-3d", 1, 5), ("deformed-cube-3d", 2, 14),
                                        ("quarter-annulus-2d", 4, 10), ("separable-nu-2d", 2, 30),
                                        ("identity-square-2d", 3, 69), ("separable-nu-2d", 2, 72)])
def test_physical_matvec_line_pair_bricks(pid, p, nel, monkeypatch):
    """Line-pair brick stencil kernel (physical.cu kernel (c): MMA rows = 4 i_1 x 2 neighbouring lines, the c4
    path): every band width KS = 2..4 (p = 1..5), d = 2 and 3, one to 18 row blocks, one and two time chunks,
    against the oracle's assembled A (solver.cpp:67-70) and the one-line kernel.  STIGA_STENCIL_REQUIRE_PAIR
    makes the launcher fail instead of falling back, so a pass means the brick kernel ran."""
    torch = pytest.importorskip("torch")
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.inputs import uniform_pm1

    prob = Problem(pid)
    ref = og.geometry_preconditioner_pieces(og.make_problem(pid), p, nel)
    A = stiga.KronSumOperator.physical(prob, p, nel)
    Ad = sp_kron(ref)
    x = uniform_pm1(A.n_dof, 8)
    yo = Ad @ x
    monkeypatch.setenv("STIGA_STENCIL_REQUIRE_PAIR", "1")
    y = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    monkeypatch.delenv("STIGA_STENCIL_REQUIRE_PAIR")
    monkeypatch.setenv("STIGA_STENCIL_NO_PAIR", "1")
    y1 = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.linalg.norm(y - y1) <= 1e-13 * np.linalg.norm(yo)
