"""Bounded-sample timing of the reference's CPU path (the oracle port) -- used ONLY by bench.py's
`cpu_baseline` leg and `--impl reference` (test infrastructure, never the product path).

One FD apply (fdsolve.cpp:155-164) is a fixed sequence of passes, each a loop over independent
units: the D^-1/2 scalings (elements), the mode products (kronop.cpp:43-73: for mode m the
`right` slab GEMMs X_b(left x n) J^T; mode 0 one GEMM over `right` columns; the time mode one GEMM over
N_s columns) and the arrowhead solve (fdsolve.cpp:24-65: independent per spatial eigen-index).  A
sample runs every pass of the oracle's own code (oracle.kronop.mode_product, oracle.fdsolve.arrowhead_solve)
on a contiguous fraction f of that pass's units and extrapolates t_pass / f_pass; the apply time is
the sum.  So a full-size c5p5 apply (710M DoF, ~2e12 flop) is timed in seconds, on the box's host
cores, with the per-unit work of the full problem.

The system mat-vec (kronop.cpp:108-115 with the reference's sparse banded factors, kronop.cpp:27-41)
is sampled the same way for the CPU GMRES estimate: n_P P-applies + n_A A-applies (gmres.cpp:42,
58, 76), Krylov vector updates excluded.
"""
import time

import numpy as np
import scipy.sparse as sp


class SampledFD:
    def __init__(self, cfg, frac, pieces=None):
        from oracle.fdsolve import ExtendedFDPreconditioner as OracleFD

        if pieces is None:
            from oracle.assembly import assemble_spatial_parametric, assemble_time_matrices

            Wt, Mt = assemble_time_matrices(cfg.p, cfg.n_el, 1.0)
            K, M = assemble_spatial_parametric(cfg.p, cfg.n_el, cfg.d)
        else:
            K, M, Wt, Mt = pieces
        self.K, self.M, self.Wt, self.Mt = K, M, Wt, Mt
        t0 = time.perf_counter()
        self.P = OracleFD.setup(K, M, Wt, Mt, 1.0, 1.0)  # D^-1/2 is sampled as its own pass below
        self.setup_s = time.perf_counter() - t0
        self.dims = list(self.P.dims)
        self.d = len(self.dims) - 1
        self.n_dof = int(np.prod(self.dims))
        self.n_s = self.n_dof // self.dims[-1]
        self.frac = frac
        rng = np.random.default_rng(cfg.seed)
        # ---- sampled units of every pass ---------------------------------------------------------
        self.passes = []  # (name, callable, fraction of the pass's units)
        ne = max(1, int(frac * self.n_dof))
        xs = rng.uniform(-1, 1, ne)
        ds = rng.uniform(0.5, 2.0, ne)
        self.passes.append(("pre_scale", lambda: ds * xs, ne / self.n_dof))
        for fwd in (True, False):
            for m in range(self.d + 1):
                self.passes.append(self._mode_pass(m, fwd, rng))
            if fwd:
                self.passes.append(self._arrow_pass(rng))
        self.passes.append(("post_scale", lambda: ds * xs, ne / self.n_dof))

    def _mode_pass(self, m, fwd, rng):
        from oracle.kronop import mode_product

        J = (self.P.transform_t if fwd else self.P.transform)[m]
        n = self.dims[m]
        left = int(np.prod(self.dims[:m]))
        right = int(np.prod(self.dims[m + 1:]))
        if right > 1:  # slab GEMMs over `right`: sample R_s whole slabs
            rs = max(1, int(round(self.frac * right)))
            dims_s, f = [left, n, rs] if m > 0 else [n, rs], rs / right
            mode = 1 if m > 0 else 0
        else:  # the time mode (slowest): one GEMM J X over left = N_s columns -> sample columns
            ls = max(1, int(round(self.frac * left)))
            dims_s, f, mode = [ls, n], ls / left, 1
        x = rng.uniform(-1, 1, int(np.prod(dims_s)))
        name = f"{'fwd' if fwd else 'bwd'}_mode{m}" if m < self.d else ("time_UtT" if fwd else "time_Ut")
        return name, (lambda: mode_product(x, dims_s, J, mode)), f

    def _arrow_pass(self, rng):
        from oracle.fdsolve import ArrowheadLU, arrowhead_solve

        lu = self.P.lu
        ls = max(1, int(round(self.frac * self.n_s)))
        sub = ArrowheadLU()
        sub.gamma, sub.nu = lu.gamma, lu.nu
        sub.lambda_s, sub.lambda_s_inv = lu.lambda_s[:ls].copy(), lu.lambda_s_inv[:ls].copy()
        sub.lambda_t, sub.zero_count, sub.g, sub.sigma = lu.lambda_t, lu.zero_count, lu.g, lu.sigma
        sub.R_inv = [r[:ls].copy() for r in lu.R_inv]
        sub.S_inv = lu.S_inv[:ls].copy()
        x = rng.uniform(-1, 1, ls * self.dims[-1])
        return "arrowhead", (lambda: arrowhead_solve(sub, x)), ls / self.n_s

    def run(self):
        """One sampled apply -> (extrapolated full-apply seconds, wall seconds of the sample, per pass)."""
        est, wall, per = 0.0, 0.0, {}
        for name, fn, f in self.passes:
            t0 = time.perf_counter()
            fn()
            dt = time.perf_counter() - t0
            wall += dt
            est += dt / f
            per[name] = per.get(name, 0.0) + dt / f
        return est, wall, per


class SampledMatvec:
    """A x = sum_t c_t (kron F_t) x with the 1D factors as SPARSE banded matrices, as the reference's
    KronFactor holds them (kronop.cpp:7-41); the identity-geometry (d+1)-term form (solver.cpp:10-30).
    Each term's mode products run on sampled slabs like SampledFD."""

    def __init__(self, fd, frac):
        from oracle.assembly import kron_sum_terms

        self.fd, self.frac = fd, frac
        self.terms = [(c, [sp.csr_matrix(f) for f in fs]) for c, fs in kron_sum_terms(fd.K, fd.M, fd.Wt, fd.Mt, 1.0, 1.0)]
        rng = np.random.default_rng(7)
        dims = fd.dims
        self.passes = []
        for ti, (c, fs) in enumerate(self.terms):
            for m, F in enumerate(fs):
                n = dims[m]
                left = int(np.prod(dims[:m]))
                right = int(np.prod(dims[m + 1:]))
                if right > 1:
                    rs = max(1, int(round(frac * right)))
                    x = rng.uniform(-1, 1, (rs, n, left))
                    f = rs / right
                    if m == 0:
                        fn = (lambda F=F, x=x: (F @ x.reshape(x.shape[0], -1).T))
                    else:
                        fn = (lambda F=F, x=x: [F @ x[b] for b in range(x.shape[0])])
                else:
                    ls = max(1, int(round(frac * left)))
                    x = rng.uniform(-1, 1, (n, ls))
                    f = ls / left
                    fn = (lambda F=F, x=x: F @ x)
                self.passes.append((f"term{ti}_mode{m}", fn, f))
        ne = max(1, int(frac * fd.n_dof))
        a, b = rng.uniform(-1, 1, ne), rng.uniform(-1, 1, ne)
        for ti in range(len(self.terms)):
            self.passes.append((f"term{ti}_accumulate", (lambda: np.add(a, 1.0 * b, out=a)), ne / fd.n_dof))

    def run(self):
        est = 0.0
        for _, fn, f in self.passes:
            t0 = time.perf_counter()
            fn()
            est += (time.perf_counter() - t0) / f
        return est


def threads_limit(n):
    """Context manager limiting the BLAS pools (OpenBLAS) to n threads (None = all)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=n)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        import os

        return os.cpu_count() or 1
