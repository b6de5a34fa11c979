"""GPU parity of the FD apply (the hot path) against the CPU oracle, through the C ABI.
Bar: ||s_gpu - s_oracle||_2 / ||s_oracle||_2 <= 1e-11 (north_star) on seeded uniform[-1,1] inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fdsolve as ofd  # noqa: E402
from oracle import kronop as okr  # noqa: E402
from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.configs import CONFIGS  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import geometry_scaling, identity_pieces  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run_pair(d, p, nel, scaled, seed=7, gamma=1.0, nu=1.0):
    pc = identity_pieces(d, p, nel)
    D = None
    if scaled:
        D = geometry_scaling(pc) * np.exp(0.3 * uniform_pm1(pc.n_dof, seed + 1))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, scaling=D, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, scaling=D)
    r = uniform_pm1(pc.n_dof, seed)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    return s, Po.apply(r), P, Po, r


@pytest.mark.parametrize("d,p,nel", [
    (1, 2, 1), (1, 1, 2), (1, 2, 5), (1, 3, 40), (1, 5, 33),         # d = 1, tiny and zero blocks
    (2, 2, 16),                                                       # c1
    (2, 1, 3), (2, 3, 8), (2, 3, 9), (2, 4, 11), (2, 2, 30),          # ragged / odd n_t (zero block)
    (3, 2, 6), (3, 3, 7), (3, 3, 12), (3, 4, 9),
    (2, 3, 64), (3, 3, 24),                                           # multi-tile sizes
])
@pytest.mark.parametrize("scaled", [False, True])
def test_fd_apply_parity(d, p, nel, scaled):
    s, so, *_ = run_pair(d, p, nel, scaled)
    assert rel(s, so) <= TOL


def test_fd_apply_nt1():
    """n_t = 1 (degenerate split, pencil.cpp:124-130): a single diagonal solve (gamma sigma + nu Lambda_s)^-1."""
    K, M = stiga.assemble_spatial_parametric(2, 5, 2)
    Wt, Mt = stiga.assemble_time_matrices(1, 1)
    P = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0)
    assert P.dims[-1] == 1 and P.time_info()["npairs"] == 0
    r = uniform_pm1(P.n_dof, 21)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(s, Po.apply(r)) <= TOL


@pytest.mark.parametrize("nel", [96, 128, 161])
def test_fd_apply_parity_large_1d_modes(nel):
    """n = 97..163 exercises WM > 1 warp-row groups and the K-chunk tail (d = 2, small time)."""
    pc = identity_pieces(2, 3, nel)
    Wt, Mt = stiga.assemble_time_matrices(3, 6)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, Wt, Mt, 1.0, 1.0, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, Wt, Mt, 1.0, 1.0)
    r = uniform_pm1(P.n_dof, 11)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(s, Po.apply(r)) <= TOL


def test_fd_apply_parity_c2_reduced_and_long_time():
    """c2's p = 3 with n_t = 258 (full c2 time direction) on a reduced spatial grid."""
    K, M = stiga.assemble_spatial_parametric(3, 20, 2)
    Wt, Mt = stiga.assemble_time_matrices(3, 256)
    P = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0)
    r = uniform_pm1(P.n_dof, 12)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(s, Po.apply(r)) <= TOL


def test_fd_apply_nu_quirk_with_product_basis():
    """nu != 1 exercises the reference's c1*c1/nu formula (fdsolve.cpp:17,128-129), whose result
    depends on the time eigenbasis; the oracle arrowhead is fed the product's exported factors."""
    K, M = stiga.assemble_spatial_parametric(2, 6, 2)
    Wt, Mt = stiga.assemble_time_matrices(2, 7)
    gamma, nu = 1.7, 2.5
    P = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, gamma, nu, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, gamma, nu)
    # rebuild the oracle's time pieces from the product's factorization
    ti = P.time_info()
    Po.time.U = P.export(2)
    Po.lu.lambda_t = list(P.export(3))
    Po.lu.g = P.export(4)
    Po.lu.S_inv = P.export(5)
    Po.lu.R_inv = [1.0 / (nu * Po.lu.lambda_s + gamma * gamma / nu * lam * lam * Po.lu.lambda_s_inv)
                   for lam in Po.lu.lambda_t]
    Po.U = [P.export(0, l) for l in range(2)]
    Po.transform = Po.U + [Po.time.U]
    Po.transform_t = [u.T.copy() for u in Po.transform]
    assert ti["zero_count"] == Po.lu.zero_count
    r = uniform_pm1(P.n_dof, 13)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(s, Po.apply(r)) <= TOL


def test_fd_apply_in_place_and_streams():
    pc = identity_pieces(2, 2, 10)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    r = torch.from_numpy(uniform_pm1(P.n_dof, 3)).cuda()
    ref = P.apply(r)
    x = r.clone()
    P.apply(x, out=x)  # aliasing allowed
    assert torch.equal(x, ref)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        y = P.apply(r)
    st.synchronize()
    assert torch.equal(y, ref)  # deterministic
    host = P.apply(r.cpu().numpy())
    assert np.array_equal(host, ref.cpu().numpy())


def test_fd_apply_errors():
    pc = identity_pieces(2, 2, 4)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    with pytest.raises(ValueError):
        P.apply(torch.zeros(P.n_dof + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        P.apply(np.zeros(3))


def test_fd_linearity_and_inverse_full_c2():
    """Full c2 size (17M DoF): size-independent properties.  On the identity geometry the FD
    preconditioner is the exact inverse of A, so A P r = r to rounding, and
    the apply is linear."""
    cfg = CONFIGS["c2"]
    pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    r = torch.from_numpy(uniform_pm1(P.n_dof, cfg.seed)).cuda()
    s = P.apply(r)
    res = torch.linalg.norm(A.apply(s) - r) / torch.linalg.norm(r)
    assert res.item() <= 1e-9
    q = torch.from_numpy(uniform_pm1(P.n_dof, 77)).cuda()
    lin = P.apply(2.0 * r - 3.0 * q) - (2.0 * s - 3.0 * P.apply(q))
    assert (torch.linalg.norm(lin) / torch.linalg.norm(s)).item() <= 1e-12


def test_kron_matvec_matches_dense():  # tests/test_kronop.cpp:62-123 through the GPU mode kernels
    rng = np.random.default_rng(11)
    x = rng.standard_normal(60)
    J = rng.standard_normal((6, 4))
    y = stiga.kron_matvec([np.eye(3), J, np.eye(5)], torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(y - okr.dense_kron_chain([np.eye(3), J, np.eye(5)]) @ x).max() <= 1e-13
    A, B, C = (rng.standard_normal((4, 4)) for _ in range(3))
    big = okr.dense_kron_chain([A, B, C])
    for j in range(64):
        e = np.zeros(64)
        e[j] = 1.0
        col = stiga.kron_matvec([A, B, C], torch.from_numpy(e).cuda()).cpu().numpy()
        assert np.abs(col - big[:, j]).max() <= 1e-13
    for n in (17, 97, 130, 258):  # the FD mode sizes
        Fs = [rng.standard_normal((n, n)) for _ in range(2)]
        xx = rng.standard_normal(n * n)
        yy = stiga.kron_matvec(Fs, torch.from_numpy(xx).cuda()).cpu().numpy()
        ref = okr.kron_matvec(Fs, xx)
        assert rel(yy, ref) <= 1e-13


@pytest.mark.parametrize("variant", ["fused", "split"])
@pytest.mark.parametrize("d,p,nel", [(1, 2, 5), (2, 3, 9), (2, 3, 30), (3, 3, 7), (1, 3, 256)])
def test_time_variants(variant, d, p, nel, monkeypatch):
    """Both time-direction paths (fused kernel / U_t^T + arrowhead + U_t passes) match the oracle."""
    monkeypatch.setenv("STIGA_TIME_VARIANT", variant)
    s, so, P, *_ = run_pair(d, p, nel, scaled=True, seed=31)
    names = [nm for nm, _ in P.launch_info()]
    assert any(nm.startswith("time_fused") for nm in names) == (variant == "fused")
    assert rel(s, so) <= TOL


@pytest.mark.parametrize("d,p,nel", [(3, 2, 64), (2, 2, 60), (1, 3, 100), (2, 3, 70), (1, 2, 72)])
@pytest.mark.parametrize("gamma,nu", [(1.0, 1.0), (1.6, 2.5)])
def test_time_resident_kernel(d, p, nel, gamma, nu, monkeypatch):
    """STIGA_TIME_KERNEL=res: the time direction on the resident-U_t persistent kernel (time_res.cu:
    one copy of U_t in smem read both ways, producer warp + mbarrier ring, arrowhead on the resident
    Z tile between named barriers), odd / even n_t (zero block), gamma, nu != 1 (the c1*c1/nu quirk),
    D^-1/2 scaled; <= 1e-11 vs the oracle, equal to the streaming time-fused kernel to rounding."""
    monkeypatch.setenv("STIGA_TIME_VARIANT", "fused")
    monkeypatch.setenv("STIGA_TIME_KERNEL", "res")
    pc = identity_pieces(d, p, nel)
    D = geometry_scaling(pc) * np.exp(0.3 * uniform_pm1(pc.n_dof, 7))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, scaling=D, device=0)
    names = [nm for nm, _ in P.launch_info()]
    assert "time_fused(res)" in names, names
    r = uniform_pm1(pc.n_dof, 12)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    if nu == 1.0:  # (nu != 1: the c1*c1/nu quirk makes the output basis dependent; the stream check below)
        Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, scaling=D)
        assert rel(s, Po.apply(r)) <= TOL
    monkeypatch.setenv("STIGA_TIME_KERNEL", "stream")
    P2 = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, gamma, nu, scaling=D, device=0)
    assert rel(s, P2.apply(torch.from_numpy(r).cuda()).cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("wn", [2, 4])
@pytest.mark.parametrize("d,p,nel", [(3, 2, 64), (2, 4, 64), (2, 3, 40), (1, 3, 66), (2, 2, 9)])
def test_time_fused_three_warp_rows(d, p, nel, wn, monkeypatch):
    """Time-fused kernel with WM = 3 warp rows (fd_time.cu: n_t = 65..72 is 9 strips = 3 x 3, the c4 /
    c5p2 shape; 96 WN threads, so the last fiber-copy round is guarded and the 6 Schur partial sums of a
    column are reduced through shared memory): odd and even n_t, S not a multiple of 3, D^-1/2 scaled,
    <= 1e-11 vs the oracle and equal to the tuned kernel to rounding."""
    monkeypatch.setenv("STIGA_TIME_VARIANT", "fused")
    monkeypatch.setenv("STIGA_FORCE_TIME_TILING", f"3,{wn},0")
    s, so, P, Po, r = run_pair(d, p, nel, scaled=True, seed=33)
    # only WM = 3 candidates exist under the forced tiling, so a fused launch is a WM = 3 launch
    assert any(nm.startswith("time_fused") for nm, _ in P.launch_info())
    assert rel(s, so) <= TOL
    monkeypatch.delenv("STIGA_FORCE_TIME_TILING")
    s2, *_ = run_pair(d, p, nel, scaled=True, seed=33)
    assert rel(s, s2) <= 1e-13


def _oracle_with_product_basis(Po, P, d, gamma=1.0, nu=1.0):
    """Rebuild the oracle's factors from the product's factorization (stiga_fd_export), so the
    comparison isolates the apply (fdsolve.cpp:155-164) from the eigensolver."""
    Po.time.U = P.export(2)
    Po.lu.lambda_t = list(P.export(3))
    Po.lu.g = P.export(4)
    Po.lu.S_inv = P.export(5)
    Po.lu.R_inv = [1.0 / (nu * Po.lu.lambda_s + gamma * gamma / nu * lam * lam * Po.lu.lambda_s_inv)
                   for lam in Po.lu.lambda_t]
    Po.U = [P.export(0, l) for l in range(d)]
    Po.transform = Po.U + [Po.time.U]
    Po.transform_t = [u.T.copy() for u in Po.transform]
    return Po


@pytest.mark.parametrize("cfg_name", ["c2", "c3", "c4", "c5p2", "c5p4", "c5p5"])
def test_fd_apply_parity_full_baseline_configs(cfg_name):
    """Full-size BASELINE configs against the oracle apply (oracle/fdsolve.py, fdsolve.cpp:155-164)
    with the ORACLE'S OWN, independent factorization (LAPACK eigensolvers vs the product's
    Householder + QL), built from the same host pieces: c2 (17.0M DoF, identity geometry, split time
    path, folded spatial products), c3 (89.4M DoF, d = 3, fused time kernel), c4 (19.3M DoF, fitted
    deformed cube with kappa(x), c(x) and the D^-1/2 geometry scaling, p = 4), c5p2 (17.0M), c5p4
    (288M, p = 4) and c5p5 (710M DoF, p = 5, the largest single-GPU config).  The p >= 4 time pencils
    meet the bar because both sides take the pairs from the Hermitian embedding (the
    reference's S^T S walk was only 1e-8 accurate at c4)."""
    from paper_1909_07309_b200.problems import Problem

    cfg = CONFIGS[cfg_name]
    if cfg.problem == "identity":
        pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
        K, M, Wt, Mt, D = pc.K, pc.M, pc.Wt, pc.Mt, geometry_scaling(pc)
    else:
        pc = Problem(cfg.problem).geometry_pieces(cfg.p, cfg.n_el, want_D=True)
        K, M, Wt, Mt, D = pc.K, pc.M, pc.Wt, pc.Mt, pc.D
    P = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D, device=0)
    r = uniform_pm1(P.n_dof, cfg.seed)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    del P
    torch.cuda.empty_cache()
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D)
    del D
    so = Po.apply(r)
    del Po, r
    assert rel(s, so) <= TOL


def test_fd_apply_parity_random_shapes():
    """Hypothesis-drawn shapes (derandomised, reproducible): d = 1..3, p = 1..5, ragged n_el, with
    and without the D^-1/2 scaling, gamma != 1 -- every tiling / strip-skipping / remainder path of
    the mode and time kernels meets the 1e-11 bar against the oracle."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=30, deadline=None, derandomize=True)
    @given(st.integers(1, 3), st.integers(1, 5), st.integers(1, 14), st.booleans(), st.floats(0.5, 3.0))
    def check(d, p, nel, scaled, gamma):
        if nel + p - 2 < 1 or (d == 3 and nel > 9):
            return
        s, so, *_ = run_pair(d, p, nel, scaled, seed=nel + 7 * p, gamma=gamma, nu=1.0)
        assert rel(s, so) <= TOL, (d, p, nel, scaled, gamma)

    check()


# ---- folded (centrosymmetric) mode products --------------------------------------------------


@pytest.mark.parametrize("d,p,nel", [
    (1, 2, 1), (1, 1, 2), (1, 2, 3), (1, 3, 40), (1, 5, 33),   # n = 1 (no split), 2, 3, odd/even
    (2, 2, 16), (2, 3, 9), (2, 4, 11), (2, 3, 64),            # c1, odd and even n, multi-chunk
    (3, 2, 6), (3, 3, 7), (3, 3, 12), (3, 4, 9), (3, 3, 24),
])
@pytest.mark.parametrize("scaled", [False, True])
def test_fd_apply_parity_folded_kernels(d, p, nel, scaled, monkeypatch):
    """STIGA_FOLD_KERNEL=force: every split spatial direction runs the folded kernels (forward fold
    x_k +- x_{n-1-k} on the B fragments, backward p +- q epilogue), <= 1e-11 vs the oracle and equal to
    the dense kernels on the same split basis to rounding."""
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "force")
    s, so, P, _, r = run_pair(d, p, nel, scaled)
    names = [nm for nm, _ in P.launch_info()]
    if P.dims[0] >= 2:
        assert any("folded" in nm for nm in names), names
    assert rel(s, so) <= TOL
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "off")
    s2, *_ = run_pair(d, p, nel, scaled)
    assert rel(s, s2) <= 1e-13


@pytest.mark.parametrize("nel", [96, 161, 254])
def test_fd_apply_parity_folded_large_modes(nel, monkeypatch):
    """n = 97 / 162 / 255 + 2: several row blocks of the folded matrices and the contraction tail."""
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "force")
    pc = identity_pieces(2, 3, nel)
    Wt, Mt = stiga.assemble_time_matrices(3, 4)
    D = np.exp(0.2 * uniform_pm1(pc.K[0].shape[0] ** 2 * Wt.shape[0], 5))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, Wt, Mt, 1.0, 1.0, scaling=D, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, Wt, Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(P.n_dof, 13)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel(s, Po.apply(r)) <= TOL


@pytest.mark.parametrize("d,p,nel", [
    (1, 3, 150), (2, 3, 96), (2, 5, 160), (2, 4, 128), (3, 2, 64), (3, 3, 60), (3, 3, 50), (2, 2, 90),
])
@pytest.mark.parametrize("scaled", [False, True])
def test_fd_apply_parity_resident_fold(d, p, nel, scaled, monkeypatch):
    """STIGA_FOLD_KERNEL=res: every split direction on the resident-factor persistent folded kernel
    (fold_res.cu: both folded factors in smem, producer warp + mbarrier ring across tiles), odd and even
    n, 4..11 strips, mode 0 (contiguous fibers) and strided modes; <= 1e-11 vs the oracle and equal to
    the streaming folded kernel to rounding."""
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "res")
    s, so, P, _, r = run_pair(d, p, nel, scaled)
    names = [nm for nm, _ in P.launch_info()]
    assert sum("folded,res" in nm for nm in names) == 2 * d, names
    assert rel(s, so) <= TOL
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "stream")
    s2, *_ = run_pair(d, p, nel, scaled)
    assert rel(s, s2) <= 1e-13


@pytest.mark.parametrize("d,p,nel", [(1, 3, 150), (2, 3, 96), (2, 5, 160), (3, 2, 64), (3, 3, 60)])
def test_fd_apply_parity_resident_fold_prescale(d, p, nel, monkeypatch):
    """The resident folded kernel with the fused D^-1/2 pre-scale (D chunks staged beside both fiber
    chunks, B fragments scaled as the fold is formed): forced with STIGA_FUSED_PRESCALE."""
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "res")
    monkeypatch.setenv("STIGA_FUSED_PRESCALE", "1")
    s, so, P, _, r = run_pair(d, p, nel, True)
    names = [nm for nm, _ in P.launch_info()]
    assert names[0].startswith("fwd_mode0(folded,res)+pre_scale"), names
    assert rel(s, so) <= TOL


@pytest.mark.parametrize("d,p,nel", [(3, 4, 9), (3, 4, 30), (2, 3, 96), (1, 5, 160), (2, 5, 160), (3, 2, 40)])
@pytest.mark.parametrize("scaled", [False, True])
def test_fd_apply_parity_dense_resident(d, p, nel, scaled, monkeypatch):
    """STIGA_DENSE_KERNEL=res with folding off and the split time path: every spatial product and both
    time GEMMs on the dense resident-factor kernel (dense_res.cu: row blocks of the factor in smem,
    persistent CTAs, producer warp + mbarrier ring; the fused D^-1/2 pre-scale when the tuner picks
    it), 1..3 row blocks, mode 0 and strided modes; <= 1e-11 vs the oracle, equal to the streaming
    kernels to rounding."""
    monkeypatch.setenv("STIGA_FOLD_KERNEL", "off")
    monkeypatch.setenv("STIGA_TIME_VARIANT", "split")
    monkeypatch.setenv("STIGA_DENSE_KERNEL", "res")
    s, so, P, _, r = run_pair(d, p, nel, scaled)
    names = [nm for nm, _ in P.launch_info()]
    assert sum("(res)" in nm for nm in names) == 2 * d + 2, names
    assert rel(s, so) <= TOL
    monkeypatch.setenv("STIGA_DENSE_KERNEL", "stream")
    s2, *_ = run_pair(d, p, nel, scaled)
    assert rel(s, s2) <= 1e-13


def test_fd_apply_parity_dense_resident_deformed(monkeypatch):
    """The config-4 kind of factors (weighted, not mirror symmetric) with the real D^-1/2 on the dense
    resident kernels."""
    from paper_1909_07309_b200.problems import Problem

    monkeypatch.setenv("STIGA_DENSE_KERNEL", "res")
    pc = Problem("deformed-cube-3d").geometry_pieces(4, 20, want_D=True)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D, device=0)
    assert any("(res)" in nm for nm, _ in P.launch_info())
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D)
    r = uniform_pm1(P.n_dof, 21)
    assert rel(P.apply(torch.from_numpy(r).cuda()).cpu().numpy(), Po.apply(r)) <= TOL


def test_fold_not_used_on_curved_geometry():
    """The A^G factors of the deformed cube are not centrosymmetric: dense kernels only."""
    from paper_1909_07309_b200.problems import Problem

    pc = Problem("deformed-cube-3d").geometry_pieces(2, 4)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=pc.D, device=0)
    assert not any("folded" in nm for nm, _ in P.launch_info())
