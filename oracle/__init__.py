"""CPU oracle for the extended-FD preconditioner hot path (TEST INFRASTRUCTURE ONLY).

This package is a numpy/scipy restatement of the reference `stiga` C++/Eigen code
under /root/reference/proj/core (which cannot be compiled here: Eigen3, doctest,
CLI11 and google-benchmark are absent -- see DESIGN.md "Oracle").  Every function
cites the reference file:line it follows.

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference`
legs of `bench.py` may import it, and only as the *checker* (or as the timed CPU
baseline).  The product path (`paper_1909_07309_b200`) never imports it and has no
CPU fallback.

Pinning: the oracle is checked against every known-answer value the
reference's own tests hold for this path (tests/test_kronop.cpp, tests/test_bspline.cpp),
the SPEC.md worked examples for pencil/fdsolve/gmres, the paper's Tables 1 and 3
(kappa_2 of U_l and U_t) and dense-inverse equivalence on small systems.  The FD
apply, time factorization and GMRES have no golden vectors in the reference suite
(their test files are empty stubs), so for those the pin is the SPEC/paper KATs plus
the dense solve.
"""
