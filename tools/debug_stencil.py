"""Runs one physical mat-vec per (problem, p, n_el) in a fresh subprocess and reports pass / CUDA failure."""
import subprocess
import sys

CASES = [(pid, p, nel) for pid in ("identity-square-2d", "identity-cube-3d") for p in (1, 2, 3, 4)
         for nel in (2, 4, 5, 6, 8)]
code = """
import sys, torch
from paper_1909_07309_b200 import stiga
from paper_1909_07309_b200.problems import Problem
from paper_1909_07309_b200.inputs import uniform_pm1
A = stiga.KronSumOperator.physical(Problem(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]))
x = torch.from_numpy(uniform_pm1(A.n_dof, 1)).cuda()
y = A.apply(x); torch.cuda.synchronize(); print('ok')
"""
for pid, p, nel in CASES:
    if pid.endswith("3d") and nel > 5:
        continue
    r = subprocess.run([sys.executable, "-c", code, pid, str(p), str(nel)], capture_output=True, text=True)
    n = nel + p - 2
    print(pid, "p", p, "nel", nel, "n", n, "n_t", nel + p - 1, "OK" if "ok" in r.stdout else "FAIL " + r.stderr.strip().splitlines()[-1][:100])
