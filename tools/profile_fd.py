"""Small driver for ncu: setup + `--applies` FD applies of a config; the LAST apply is bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures exactly one apply, in launch
order (P.launch_info() names them)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.configs import CONFIGS  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--applies", type=int, default=2)
ap.add_argument("--names-out", default=None)
a = ap.parse_args()
cfg = CONFIGS[a.config]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import problem_pieces  # noqa: E402

pc, D = problem_pieces(cfg)
P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
r = torch.from_numpy(uniform_pm1(P.n_dof, cfg.seed)).cuda()
s = torch.empty_like(r)
for _ in range(max(0, a.applies - 1)):
    P.apply(r, out=s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
P.apply(r, out=s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
if a.names_out:
    json.dump({"config": cfg.name, "n_dof": P.n_dof, "launches": P.launch_info()}, open(a.names_out, "w"))
print("ok", a.config, P.n_dof, P.launch_info())
