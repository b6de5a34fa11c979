"""Spatial / temporal pencil factorizations (oracle).  Follows /root/reference/proj/core/src/pencil.cpp."""
import numpy as np
import scipy.linalg as sla


def spd_generalized_eig(K, M):
    """pencil.cpp:12-21: K U = M U Lambda, U^T M U = I, ascending (LAPACK dsygvd here,
    Eigen GeneralizedSelfAdjointEigenSolver in the reference; the FD output is basis invariant)."""
    K = np.asarray(K, dtype=np.float64)
    M = np.asarray(M, dtype=np.float64)
    if K.shape[0] != K.shape[1] or M.shape != K.shape:
        raise ValueError("spd_generalized_eig: shape mismatch")
    try:
        lam, U = sla.eigh(K, M)
    except np.linalg.LinAlgError as e:
        raise RuntimeError("spd_generalized_eig: mass matrix not SPD") from e
    return U, lam


class SkewPencilEig:
    def __init__(self, U, lam, zero_count):
        self.U, self.lam, self.zero_count = U, lam, zero_count


def _reduce_skew(W, M):
    """pencil.cpp:30-44: shape / skewness checks, Cholesky of M, S = L^-1 W L^-T skew-symmetrized."""
    W = np.asarray(W, dtype=np.float64)
    M = np.asarray(M, dtype=np.float64)
    n = W.shape[0]
    if W.shape != (n, n) or M.shape != (n, n):
        raise ValueError("skew_pencil_eig: shape mismatch")
    if n == 0:
        return None, None, None
    wmax = np.abs(W).max()
    if np.abs(W + W.T).max() > 1e-13 * max(wmax, 1.0):
        raise RuntimeError("skew_pencil_eig: matrix is not skew-symmetric (assembly bug)")
    try:
        L = np.linalg.cholesky(M)
    except np.linalg.LinAlgError as e:
        raise RuntimeError("skew_pencil_eig: mass matrix not SPD") from e
    S = sla.solve_triangular(L, W, lower=True)
    S = sla.solve_triangular(L, S.T, lower=True).T
    S = 0.5 * (S - S.T)
    return n, L, S


def skew_pencil_eig(W, M):
    """Real-block eigendecomposition of the skew pencil (W, M) with the contract of
    pencil.cpp:23-95: U^T M U = I, U^T W U = blockdiag([[0, lam_j], [-lam_j, 0]], 0..), pair columns
    (v, q) in ascending lam, zero columns last.

    Deliberate deviation: the pairs come from the Hermitian eigenproblem of iS through
    its real symmetric embedding (`_embedding_pairs`), not from the eigenvectors of S^T S.  The
    reference's S^T S walk (restated in `skew_pencil_eig_walk`) squares the conditioning: at p = 4,
    n_el = 64 (config 4) its U^T M U - I is 1e-8, the embedding's 5e-15; at p = 3, n_el = 256
    (config 2) the walk fails outright ("eigenvalue pairing failed")."""
    n, L, S = _reduce_skew(W, M)
    if n is None:
        return SkewPencilEig(np.zeros((0, 0)), [], 0)
    mu, Q = np.linalg.eigh(S.T @ S)  # only to count / seed the zero columns (pencil.cpp:50-52, 72-76)
    mu = np.maximum(mu, 0.0)
    zero_tol = 1e-12 * max(mu[n - 1], 1.0)
    lam_out, pair_cols = _embedding_pairs(S, zero_tol)
    nz = n - 2 * len(lam_out)
    if nz < 0 or nz > int(np.sum(mu <= zero_tol)) + 1:
        raise RuntimeError("skew_pencil_eig: eigenvalue pairing failed")
    B = np.column_stack(pair_cols) if pair_cols else np.zeros((n, 0))
    zero_cols = []
    for k in range(nz):  # null vectors of S, orthogonal to every pair column (two passes)
        q = Q[:, k].copy()
        for _ in range(2):
            q -= B @ (B.T @ q)
            for c in zero_cols:
                q -= c.dot(q) * c
        zero_cols.append(q / np.linalg.norm(q))
    Ublk = np.column_stack(pair_cols + zero_cols)
    U = sla.solve_triangular(L.T, Ublk, lower=False)  # pencil.cpp:93
    return SkewPencilEig(U, lam_out, nz)


def skew_pencil_eig_walk(W, M):
    """pencil.cpp:23-95 as written: Cholesky reduction, eig of S^T S, pair walk, zero columns last.
    Kept as the restatement of the reference algorithm (tests pin where it fails or loses accuracy);
    `skew_pencil_eig` is the one the oracle uses."""
    n, L, S = _reduce_skew(W, M)
    if n is None:
        return SkewPencilEig(np.zeros((0, 0)), [], 0)
    C = S.T @ S
    mu, Q = np.linalg.eigh(C)
    mu = np.maximum(mu, 0.0)
    mu_max = max(mu[n - 1], 1.0)
    zero_tol = 1e-12 * mu_max
    zero_cols, pair_cols, lam_out = [], [], []
    cluster, cluster_mu = [], -1.0
    for k in range(n):
        q = Q[:, k].copy()
        if mu[k] > cluster_mu + zero_tol:
            cluster = []
            cluster_mu = mu[k]
        for c in cluster:
            q -= c.dot(q) * c
        nrm = np.linalg.norm(q)
        if nrm < 1e-6:
            continue
        q /= nrm
        if mu[k] <= zero_tol:
            zero_cols.append(q)
            cluster.append(q)
            continue
        lam = np.sqrt(mu[k])
        v = S @ q / lam
        lam_out.append(lam)
        pair_cols += [v, q]
        cluster += [q, v]
    if len(pair_cols) + len(zero_cols) != n:
        raise RuntimeError("skew_pencil_eig: eigenvalue pairing failed")  # pencil.cpp:86-87
    Ublk = np.column_stack(pair_cols + zero_cols)
    U = sla.solve_triangular(L.T, Ublk, lower=False)
    return SkewPencilEig(U, lam_out, len(zero_cols))


def _embedding_pairs(S, zero_tol_mu):
    """Real pairs (v, q) with S q = lam v, S v = -lam q from the real symmetric embedding
    E = [[0, -S], [S, 0]] of the Hermitian iS: E [x; y] = lam [x; y]  <=>  S x = lam y, -S y = lam x,
    so q = sqrt(2) x, v = sqrt(2) y.  Every positive eigenvalue of E is double (z and Jz,
    J [x; y] = [-y; x]); the pairs are built by pivoted Gram-Schmidt over each cluster's J-invariant
    eigenspace, orthogonalising every new z and Jz against ALL accepted vectors (two passes), so
    distinct pairs whose eigenvalues are closer than the eigensolver can separate stay exactly
    orthonormal (their mixing only perturbs U^T W U by gap x mixing ~ eps)."""
    n = S.shape[0]
    E = np.zeros((2 * n, 2 * n))
    E[:n, n:] = -S
    E[n:, :n] = S
    w, V = np.linalg.eigh(E)
    lam_tol = np.sqrt(zero_tol_mu)
    pos = [k for k in range(2 * n) if w[k] > lam_tol]
    lam_max = max(w[-1], 1.0)
    clusters, cur = [], []
    for k in pos:
        if cur and w[k] - w[cur[-1]] > 1e-8 * lam_max:
            clusters.append(cur)
            cur = []
        cur.append(k)
    if cur:
        clusters.append(cur)
    basis = []

    def project(r):
        for _ in range(2):
            for b in basis:
                r -= b.dot(r) * b
        return r

    pairs = []
    for cl in clusters:
        cand = [V[:, k].copy() for k in cl]
        for _ in range(len(cl) // 2):
            best, bnorm = None, -1.0
            for c in cand:
                r = project(c.copy())
                nr = np.linalg.norm(r)
                if nr > bnorm:
                    best, bnorm = r, nr
            z = project(best / bnorm)
            z /= np.linalg.norm(z)
            basis.append(z)
            jz = project(np.concatenate([-z[n:], z[:n]]))
            jz /= np.linalg.norm(jz)
            basis.append(jz)
            lam = z.dot(E @ z)
            pairs.append((lam, np.sqrt(2.0) * z[n:], np.sqrt(2.0) * z[:n]))
    pairs.sort(key=lambda t: t[0])
    lam_out = [t[0] for t in pairs]
    cols = []
    for _, v, q in pairs:
        cols += [v, q]
    return lam_out, cols


_robust_pairs = _embedding_pairs  # name used by round-1 tests


class TimeFactorization:
    """pencil.hpp:40-52."""

    def __init__(self, U, lam, zero_count, g, sigma, r, rho):
        self.U, self.lam, self.zero_count = U, lam, zero_count
        self.g, self.sigma, self.r, self.rho = g, sigma, r, rho

    @property
    def size(self):
        return self.U.shape[0]

    def delta(self):
        """pencil.cpp:97-110."""
        n = self.size
        D = np.zeros((n, n))
        for j, lam in enumerate(self.lam):
            D[2 * j, 2 * j + 1] = lam
            D[2 * j + 1, 2 * j] = -lam
        if n > 1:
            D[: n - 1, n - 1] = self.g
            D[n - 1, : n - 1] = -self.g
        D[n - 1, n - 1] = self.sigma
        return D


def time_factorization(Wt, Mt):
    """pencil.cpp:112-165."""
    W = np.asarray(Wt, dtype=np.float64)
    M = np.asarray(Mt, dtype=np.float64)
    n = W.shape[0]
    if M.shape[0] != n or n < 1:
        raise ValueError("time_factorization: shape mismatch")
    U = np.zeros((n, n))
    if n == 1:
        rho = 1.0 / np.sqrt(M[0, 0])
        U[0, 0] = rho
        return TimeFactorization(U, [], 0, np.zeros(0), rho * W[0, 0] * rho, np.zeros(0), rho)
    W0, M0 = W[: n - 1, : n - 1], M[: n - 1, : n - 1]
    w, m = W[: n - 1, n - 1], M[: n - 1, n - 1]
    skew = skew_pencil_eig(W0, M0)
    try:
        c = sla.cho_factor(M0, lower=True)
    except np.linalg.LinAlgError as e:
        raise RuntimeError("time_factorization: leading time mass block not SPD") from e
    v = sla.cho_solve(c, -m)
    q = np.concatenate([v, [1.0]])
    s = np.sqrt(q.dot(M @ q))
    r = v / s
    rho = 1.0 / s
    U[: n - 1, : n - 1] = skew.U
    U[: n - 1, n - 1] = r
    U[n - 1, n - 1] = rho
    g = skew.U.T @ (W0 @ r + w * rho)
    rr = np.concatenate([r, [rho]])
    sigma = rr.dot(W @ rr)
    return TimeFactorization(U, list(skew.lam), skew.zero_count, g, sigma, r, rho)


def cond2(A):
    """pencil.cpp:185-205 (diagnostic; used by the paper-table pins)."""
    sv = np.linalg.svd(np.asarray(A), compute_uv=False)
    if sv[-1] == 0.0:
        raise RuntimeError("cond2: singular matrix")
    return sv[0] / sv[-1]
