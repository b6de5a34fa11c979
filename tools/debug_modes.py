import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_07309_b200 import stiga
from oracle import kronop as okr, fdsolve as ofd
from paper_1909_07309_b200.problems import identity_pieces
from paper_1909_07309_b200.inputs import uniform_pm1
rng = np.random.default_rng(0)
for n in (8, 13, 16, 20, 31, 32, 33, 47, 48, 49, 63, 64, 65, 66, 97, 130, 257):
    F = [rng.standard_normal((n, n)), rng.standard_normal((5, 5))]
    x = rng.standard_normal(n * 5)
    y = stiga.kron_matvec(F, torch.from_numpy(x).cuda()).cpu().numpy()
    e0 = np.linalg.norm(y - okr.kron_matvec(F, x)) / np.linalg.norm(y)
    F2 = [rng.standard_normal((5, 5)), rng.standard_normal((n, n))]
    y2 = stiga.kron_matvec(F2, torch.from_numpy(x).cuda()).cpu().numpy()
    e1 = np.linalg.norm(y2 - okr.kron_matvec(F2, x)) / np.linalg.norm(y2)
    F3 = [rng.standard_normal((70, 70)), rng.standard_normal((n, n))]
    x3 = rng.standard_normal(n * 70)
    y3 = stiga.kron_matvec(F3, torch.from_numpy(x3).cuda()).cpu().numpy()
    e2 = np.linalg.norm(y3 - okr.kron_matvec(F3, x3)) / np.linalg.norm(y3)
    print(f"n={n:4d} mode0 {e0:.1e} mode1(L=5) {e1:.1e} mode1(L=70) {e2:.1e}")
for (d, p, nel) in [(1, 3, 62), (1, 3, 63), (1, 3, 64), (2, 3, 30), (2, 3, 64)]:
    pc = identity_pieces(d, p, nel)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    r = uniform_pm1(P.n_dof, 7)
    s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    so = Po.apply(r)
    print(d, p, nel, P.dims, np.linalg.norm(s - so) / np.linalg.norm(so))
