"""Device-side setup: Lambda_s / S^-1 on the device (bit-identical to the host loop of
fdsolve.cpp:91-136), D^-1/2 from a device D, cuSOLVER eigensolves for the pencils, and the geometry
scaling D = diag(A)/diag(A~) (solver.cpp:138-142, kronop.cpp:117-131) formed on the device."""
import numpy as np
import pytest
import torch

from oracle import fdsolve as ofd
from paper_1909_07309_b200 import stiga
from paper_1909_07309_b200.inputs import uniform_pm1
from paper_1909_07309_b200.problems import Problem, geometry_scaling, identity_pieces, kron_sum_diagonal

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


SHAPES = [(1, 3, 40), (2, 2, 16), (2, 3, 9), (2, 4, 11), (3, 2, 6), (3, 3, 7), (3, 4, 9), (2, 3, 64)]


@pytest.mark.parametrize("d,p,nel", SHAPES)
@pytest.mark.parametrize("gamma,nu", [(1.0, 1.0), (1.7, 2.5)])
def test_device_schur_bit_identical(d, p, nel, gamma, nu):
    pc = identity_pieces(d, p, nel)
    Ph = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, device=0)
    Pd = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, device=0, device_schur=True)
    assert np.array_equal(Ph.export(5), Pd.export(5))
    r = torch.from_numpy(uniform_pm1(pc.n_dof, 3)).cuda()
    assert rel(Pd.apply(r).cpu().numpy(), Ph.apply(r).cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("d,p,nel", [(2, 3, 9), (3, 2, 6)])
def test_device_scaling(d, p, nel):
    pc = identity_pieces(d, p, nel)
    D = geometry_scaling(pc) * np.exp(0.3 * uniform_pm1(pc.n_dof, 11))
    Ph = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
    Pd = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=torch.from_numpy(D).cuda(),
                                              device=0, device_schur=True)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(pc.n_dof, 4)
    sd = Pd.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(sd, Ph.apply(torch.from_numpy(r).cuda()).cpu().numpy()) <= 1e-14
    assert rel(sd, Po.apply(r)) <= TOL
    Dbad = D.copy()
    Dbad[7] = -1.0
    with pytest.raises(ValueError) as e:
        stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=torch.from_numpy(Dbad).cuda(),
                                             device=0)
    assert "strictly positive" in str(e.value)


@pytest.mark.parametrize("d,p,nel", SHAPES + [(2, 3, 128), (3, 3, 24), (1, 5, 33)])
@pytest.mark.parametrize("scaled", [False, True])
def test_cusolver_eigensolver_parity(d, p, nel, scaled):
    """Every eigenproblem of the setup on cuSOLVER (syevd): the apply meets the 1e-11 bar against the
    oracle's LAPACK factorization (the bases differ; the FD output is basis-invariant)."""
    pc = identity_pieces(d, p, nel)
    D = geometry_scaling(pc) * np.exp(0.3 * uniform_pm1(pc.n_dof, 5)) if scaled else None
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0,
                                             device_schur=True, eig="cusolver")
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(pc.n_dof, 6)
    assert rel(P.apply(torch.from_numpy(r).cuda()).cpu().numpy(), Po.apply(r)) <= TOL


def test_cusolver_deformed_cube():
    pr = Problem("deformed-cube-3d")
    pc = pr.geometry_pieces(3, 8, want_D=True)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D, device=0,
                                             device_schur=True, eig="cusolver")
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D)
    r = uniform_pm1(P.n_dof, 8)
    assert rel(P.apply(torch.from_numpy(r).cuda()).cpu().numpy(), Po.apply(r)) <= TOL


@pytest.mark.parametrize("d,p,nel", [(2, 3, 9), (3, 2, 6)])
def test_kronsum_diagonal_device_bit_identical(d, p, nel):
    pc = identity_pieces(d, p, nel)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.3, 0.7)
    assert np.array_equal(A.diagonal_device().cpu().numpy(), A.diagonal())


@pytest.mark.parametrize("pid,p,nel", [("deformed-cube-3d", 2, 4), ("quarter-annulus-2d", 3, 6), ("separable-nu-2d", 2, 5)])
def test_geometry_scaling_device_bit_identical(pid, p, nel):
    pr = Problem(pid)
    pc = pr.geometry_pieces(p, nel, want_D=False)
    A = stiga.KronSumOperator.physical(pr, p, nel, device=0)
    assert np.array_equal(A.diagonal_device().cpu().numpy(), A.diagonal())
    At = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    D = stiga.geometry_scaling_device(A, At).cpu().numpy()
    Dh = A.diagonal() / kron_sum_diagonal(stiga.kron_sum_terms(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0))
    assert np.array_equal(D, Dh)
