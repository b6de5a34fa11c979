import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_07309_b200 import stiga
from oracle import fdsolve as ofd
from paper_1909_07309_b200.problems import identity_pieces
from paper_1909_07309_b200.inputs import uniform_pm1
pc = identity_pieces(1, 3, 14)
P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
r = uniform_pm1(P.n_dof, 7)
s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
if os.environ.get("STIGA_DEBUG_ARROW"):
    U = P.export(0, 0); Ut = P.export(2)
    X = r.reshape(P.dims[1], P.dims[0]).T  # (n_s, n_t)
    so = ((U @ (U.T @ X)) @ Ut @ Ut.T).T.reshape(-1)
    so = (U @ ((U.T @ X) @ (Ut @ Ut.T).T)).T.reshape(-1)
else:
    so = Po.apply(r)
print(os.environ.get("STIGA_FORCE_TIME_TILING"), os.environ.get("STIGA_DEBUG_ARROW"), P.dims, "%.2e" % (np.linalg.norm(s - so) / np.linalg.norm(so)))
