"""ncu driver for the space-time mat-vec (c4 physical by default, Kronecker-sum form for identity configs): run
`--applies` mat-vecs, bracket the last one with cudaProfilerStart/Stop."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.configs import CONFIGS  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import Problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--applies", type=int, default=3)
a = ap.parse_args()
cfg = CONFIGS[a.config]
t = time.time()
if cfg.problem == "identity":  # Kronecker-sum (banded) form of the space-time system
    from paper_1909_07309_b200.problems import identity_pieces

    pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
else:
    A = stiga.KronSumOperator.physical(Problem(cfg.problem), cfg.p, cfg.n_el)
torch.cuda.synchronize()
print("assembly_s", time.time() - t)
x = torch.from_numpy(uniform_pm1(A.n_dof, cfg.seed)).cuda()
for _ in range(max(0, a.applies - 1)):
    y = A.apply(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    y = A.apply(x)
e1.record()
torch.cuda.synchronize()
print("matvec_ms", e0.elapsed_time(e1) / 5)
torch.cuda.cudart().cudaProfilerStart()
y = A.apply(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", a.config, A.n_dof)
