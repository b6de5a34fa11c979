"""CPU checks of the product library: it loads, exports every symbol include/stiga_gpu.h declares,
and its host-side setup (1D assembly, pencils, Schur diagonal) matches the oracle.  No GPU compute."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import assembly as oasm
from oracle import fdsolve as ofd
from oracle import pencil as open_
from paper_1909_07309_b200 import _lib, stiga

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "stiga_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stiga_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes signature table"
    assert L.stiga_abi_version() == 101


def test_compute_without_device_fails_loudly():
    if stiga.device_count() > 0:
        pytest.skip("a device is present")
    pc_K, pc_M = stiga.assemble_spatial_parametric(2, 4, 1)
    W, M = stiga.assemble_time_matrices(2, 4)
    with pytest.raises(_lib.StigaError):
        stiga.ExtendedFDPreconditioner.setup(pc_K, pc_M, W, M, 1.0, 1.0, device=0)


@pytest.mark.parametrize("p,nel", [(1, 1), (1, 3), (2, 4), (3, 8), (4, 5), (5, 7)])
def test_assembly_matches_oracle(p, nel):
    W, M = stiga.assemble_time_matrices(p, nel, 1.0)
    Wo, Mo = oasm.assemble_time_matrices(p, nel, 1.0)
    assert np.abs(W - Wo).max() <= 1e-15 and np.abs(M - Mo).max() <= 1e-15
    if nel + p - 2 >= 1:
        K, Ms = stiga.assemble_spatial_parametric(p, nel, 1)
        Ko, Mso = oasm.assemble_spatial_parametric(p, nel, 1)
        assert np.abs(K[0] - Ko[0]).max() <= 1e-12 * np.abs(Ko[0]).max()
        assert np.abs(Ms[0] - Mso[0]).max() <= 1e-15
    w = np.linspace(0.5, 2.0, nel)
    A = stiga.assemble_univariate(p, nel, True, p + 1, 0, 0, w)
    from oracle.bspline import SplineSpace1D, gauss_rule
    sp = SplineSpace1D.temporal(p, nel)
    Ao = oasm.assemble_univariate(sp, gauss_rule(sp.kv, p + 1), 0, 0, element_weights=w)
    assert np.abs(A - Ao).max() <= 1e-15


def test_assembly_errors():
    with pytest.raises(ValueError):
        stiga.assemble_time_matrices(2, 4, 0.0)
    with pytest.raises(ValueError):
        stiga.space_dim(0, 4)
    with pytest.raises(RuntimeError):  # std::runtime_error for non-positive weights (assembly.cpp:62-63)
        stiga.assemble_univariate(2, 4, True, 3, 0, 0, -np.ones(4))


def _host_handle(d, p, nel, gamma=1.0, nu=1.0, scaling=None):
    K, M = stiga.assemble_spatial_parametric(p, nel, d)
    W, Mt = stiga.assemble_time_matrices(p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, gamma, nu, scaling=scaling, device=-1)
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, gamma, nu, scaling=scaling)
    return P, Po, (K, M, W, Mt)


@pytest.mark.parametrize("d,p,nel", [(1, 1, 2), (2, 2, 8), (2, 3, 9), (3, 3, 5), (1, 5, 16), (2, 2, 64), (2, 3, 256)])
def test_host_setup_matches_oracle(d, p, nel):
    P, Po, (K, M, W, Mt) = _host_handle(d, p, nel)
    assert P.dims == Po.dims and P.n_dof == Po.n_dof
    for l in range(d):
        U, lam = P.export(0, l), P.export(1, l)
        assert np.abs(lam - Po.lam[l]).max() <= 1e-11 * max(1.0, lam.max())
        assert np.abs(U.T @ M[l] @ U - np.eye(len(lam))).max() <= 1e-11
        assert np.linalg.norm(K[l] @ U - M[l] @ U @ np.diag(lam)) <= 1e-10 * np.linalg.norm(K[l])
    ti = P.time_info()
    tf = Po.time
    assert ti["npairs"] == len(tf.lam) and ti["zero_count"] == tf.zero_count
    assert ti["sigma"] == pytest.approx(tf.sigma, rel=1e-11) and ti["rho"] == pytest.approx(tf.rho, rel=1e-12)
    if tf.lam:
        assert np.abs(P.export(3) - np.array(tf.lam)).max() <= 1e-10 * max(1.0, max(tf.lam))
    Ut = P.export(2)
    n = Ut.shape[0]
    assert np.abs(Ut.T @ Mt @ Ut - np.eye(n)).max() <= 1e-10
    # U_t^T W_t U_t = Delta_t with the product's own g / sigma (eq:time_eig_2)
    g = P.export(4)
    Dt = open_.TimeFactorization(Ut, list(P.export(3)), ti["zero_count"], g, ti["sigma"], None, ti["rho"]).delta()
    assert np.linalg.norm(W @ Ut - Mt @ Ut @ Dt) <= 1e-8 * np.linalg.norm(W)
    # S^-1 is basis invariant at nu = 1 (depends on g_a^2 + g_b^2 per pair)
    assert np.abs(P.export(5) - Po.lu.S_inv).max() <= 1e-11 * np.abs(Po.lu.S_inv).max()


def test_host_setup_errors():
    K, M = stiga.assemble_spatial_parametric(2, 4, 1)
    W, Mt = stiga.assemble_time_matrices(2, 4)
    with pytest.raises(ValueError):
        stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 0.0, 1.0, device=-1)
    with pytest.raises(ValueError):
        stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 0.0, device=-1)
    with pytest.raises(ValueError):
        stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=np.ones(7), device=-1)
    with pytest.raises(ValueError):
        stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=np.zeros(4 * 5), device=-1)
    with pytest.raises(RuntimeError):  # non-SPD mass -> runtime_error (pencil.cpp:17-18)
        stiga.ExtendedFDPreconditioner.setup(K, [-M[0]], W, Mt, 1.0, 1.0, device=-1)
    P = stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, device=-1)
    with pytest.raises(ValueError):  # host-only handle cannot apply
        P.apply(np.zeros(P.n_dof))


@pytest.mark.parametrize("p,nel", [(2, 16), (3, 256), (3, 96), (4, 64), (2, 64), (4, 128), (5, 160)])
def test_host_time_factorization_accuracy_baseline_pencils(p, nel):
    """The product's own eigensolver (Householder + QL on the Hermitian embedding, host/pencil.cpp)
    reaches the oracle's accuracy on every BASELINE time pencil: U_t^T M_t U_t = I and
    U_t^T W_t U_t = Delta_t to ~1e-14 (p = 4 at config 4 was 2.5e-8 with the S^T S walk)."""
    K, M = stiga.assemble_spatial_parametric(p, 4, 1)
    W, Mt = stiga.assemble_time_matrices(p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, device=-1)
    ti = P.time_info()
    Ut = P.export(2)
    n = Ut.shape[0]
    Dt = open_.TimeFactorization(Ut, list(P.export(3)), ti["zero_count"], P.export(4), ti["sigma"], None,
                                 ti["rho"]).delta()
    assert np.abs(Ut.T @ Mt @ Ut - np.eye(n)).max() <= 1e-13
    assert np.abs(Ut.T @ W @ Ut - Dt).max() <= 1e-13 * np.abs(Dt).max()
    tf = open_.time_factorization(W, Mt)
    assert np.abs(P.export(3) - np.array(tf.lam)).max() <= 1e-12 * max(tf.lam)
