import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_07309_b200 import stiga
from oracle import fdsolve as ofd
from paper_1909_07309_b200.problems import identity_pieces
from paper_1909_07309_b200.inputs import uniform_pm1
for (d, p, nel) in [(1, 3, 62), (1, 3, 63), (1, 3, 64), (1, 3, 125), (1,3,126)]:
    pc = identity_pieces(d, p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    r = uniform_pm1(P.n_dof, 7)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    so = Po.apply(r)
    print(os.environ.get("STIGA_FORCE_TIME_TILING"), d, p, nel, P.dims, "%.2e" % (np.linalg.norm(s - so) / np.linalg.norm(so)))
