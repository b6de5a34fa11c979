"""Generates the committed golden fixtures in tests/golden/ from the CPU oracle (oracle/), which is
itself pinned to the reference's known-answer tests (tests/test_oracle_kats.py).  The reference
C++ cannot be built here (Eigen3 absent), so these are oracle vectors; they freeze the parity
target so the GPU tests on the box do not depend on scipy/LAPACK versions.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.assembly import assemble_spatial_parametric, assemble_time_matrices, kron_sum_terms  # noqa: E402
from oracle.fdsolve import ExtendedFDPreconditioner  # noqa: E402
from oracle.gmres import gmres  # noqa: E402
from oracle.kronop import KronSumOperator  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402

CASES = [  # (name, d, p, n_el, scaled, seed)
    ("c1", 2, 2, 16, False, 1),
    ("c1_scaled", 2, 2, 16, True, 11),
    ("d1_p3_n9_zero_block", 1, 3, 9, True, 12),
    ("d3_p2_n5", 3, 2, 5, True, 13),
]


def main():
    out = os.path.dirname(os.path.abspath(__file__))
    for name, d, p, nel, scaled, seed in CASES:
        W, Mt = assemble_time_matrices(p, nel, 1.0)
        K, M = assemble_spatial_parametric(p, nel, d)
        n = K[0].shape[0] ** d * W.shape[0]
        D = np.exp(0.3 * uniform_pm1(n, seed + 100)) if scaled else None
        P = ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=D)
        r = uniform_pm1(n, seed)
        s = P.apply(r)
        A = KronSumOperator(P.dims, kron_sum_terms(K, M, W, Mt, 1.0, 1.0))
        x, rep = gmres(A.apply, P.apply, r, tol=1e-8, max_krylov=100, restart=50)
        np.savez_compressed(os.path.join(out, f"{name}.npz"), d=d, p=p, n_el=nel, seed=seed,
                            scaling=D if D is not None else np.zeros(0), r=r, s=s, x=x,
                            iterations=rep.iterations, residual_history=np.array(rep.residual_history))
        print(name, n, rep.iterations)


if __name__ == "__main__":
    main()
