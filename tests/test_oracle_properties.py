"""Property-based checks of the oracle restatement (hypothesis, CPU): the mode-product / Kronecker
kernels against dense Kronecker products on random shapes, and the FD preconditioner as the exact
inverse of the space-time Kronecker-sum system on random small parametric problems
(the reference's own KATs are in test_oracle_kats.py)."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import assembly as oasm
from oracle import fdsolve as ofd
from oracle import kronop as okr


@settings(max_examples=40, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 5), st.integers(1, 5)), min_size=1, max_size=4), st.integers(0, 2**31 - 1))
def test_kron_matvec_matches_dense(shapes, seed):
    rng = np.random.default_rng(seed)
    factors = [rng.standard_normal((m, n)) for m, n in shapes]
    x = rng.standard_normal(int(np.prod([n for _, n in shapes])))
    y = okr.kron_matvec(factors, x)
    yd = okr.dense_kron_chain(factors) @ x
    assert np.allclose(y, yd, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(yd).max()))


@settings(max_examples=40, deadline=None)
@given(st.lists(st.integers(1, 5), min_size=1, max_size=4), st.integers(0, 2**31 - 1), st.data())
def test_mode_product_is_one_kron_factor(dims, seed, data):
    rng = np.random.default_rng(seed)
    mode = data.draw(st.integers(0, len(dims) - 1))
    m = data.draw(st.integers(1, 5))
    J = rng.standard_normal((m, dims[mode]))
    x = rng.standard_normal(int(np.prod(dims)))
    y, new_dims = okr.mode_product(x, dims, J, mode)
    factors = [J if k == mode else np.eye(n) for k, n in enumerate(dims)]
    assert new_dims == [m if k == mode else n for k, n in enumerate(dims)]
    assert np.allclose(y, okr.dense_kron_chain(factors) @ x, rtol=1e-12, atol=1e-12)


@settings(max_examples=15, deadline=None)
@given(st.integers(1, 2), st.integers(1, 3), st.integers(2, 5), st.floats(0.5, 2.0), st.integers(0, 2**31 - 1))
def test_fd_is_exact_inverse_of_kron_sum(d, p, nel, gamma, seed):
    """At nu = 1 (where the reference's c1*c1/nu term is exact, fdsolve.cpp:17) the extended FD
    preconditioner inverts gamma W_t (x) M_s + M_t (x) K_s for any gamma."""
    W, Mt = oasm.assemble_time_matrices(p, nel, 1.0)
    K, M = oasm.assemble_spatial_parametric(p, nel, d)
    dims = [k.shape[0] for k in K] + [W.shape[0]]
    A = okr.KronSumOperator(dims, oasm.kron_sum_terms(K, M, W, Mt, gamma, 1.0))
    P = ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, gamma, 1.0)
    r = np.random.default_rng(seed).uniform(-1, 1, A.n_dof)
    s = P.apply(r)
    assert np.linalg.norm(A.apply(s) - r) <= 1e-9 * np.linalg.norm(r)
