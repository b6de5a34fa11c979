"""GPU debugging aid: FD apply parity vs the oracle with the folded kernels forced on / off, for one
(d, p, n_el) shape (usage: python tools/debug_fold.py d p n_el [time_nel])."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import fdsolve as ofd  # noqa: E402
from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import geometry_scaling, identity_pieces  # noqa: E402

d, p, nel = (int(x) for x in sys.argv[1:4])
pc = identity_pieces(d, p, nel)
if len(sys.argv) > 4:
    pc.Wt, pc.Mt = stiga.assemble_time_matrices(p, int(sys.argv[4]))
nd = pc.K[0].shape[0] ** d * pc.Wt.shape[0]
for scaled in (False, True):
    D = np.exp(0.3 * uniform_pm1(nd, 32)) if scaled else None
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(nd, 31)
    so = Po.apply(r)
    out = {}
    for mode in ("off", "force"):
        for tv in ("fused", "split"):
            os.environ["STIGA_FOLD_KERNEL"] = mode
            os.environ["STIGA_TIME_VARIANT"] = tv
            P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
            s = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
            out[(mode, tv)] = s
            print(f"scaled={scaled} fold={mode} time={tv}: rel err {np.linalg.norm(s - so) / np.linalg.norm(so):.3e}",
                  [nm for nm, _ in P.launch_info()])
    a, b = out[("off", "fused")], out[("force", "fused")]
    print("  fold vs dense:", np.linalg.norm(a - b) / np.linalg.norm(a))
