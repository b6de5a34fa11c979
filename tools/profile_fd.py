"""Small driver for ncu: setup + `--applies` FD applies (+ optional system mat-vec) of a config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.configs import CONFIGS  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import geometry_scaling, identity_pieces  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--applies", type=int, default=2)
ap.add_argument("--matvec", action="store_true")
a = ap.parse_args()
cfg = CONFIGS[a.config]
pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=geometry_scaling(pc), device=0)
r = torch.from_numpy(uniform_pm1(P.n_dof, cfg.seed)).cuda()
s = torch.empty_like(r)
for _ in range(a.applies):
    P.apply(r, out=s)
if a.matvec:
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    for _ in range(a.applies):
        A.apply(r, out=s)
torch.cuda.synchronize()
print("ok", a.config, P.n_dof, P.launches(), "launches per apply")
