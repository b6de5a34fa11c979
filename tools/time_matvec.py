"""Times the space-time system mat-vec (KronSumOperator::apply) on identity-geometry configs and
checks the fused kernels against the banded-pass path (STIGA_MATVEC_PASSES=1 in a child process).

    python tools/time_matvec.py c3 c5p5 ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(cfg_name, out_path):
    import numpy as np
    import torch

    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.configs import CONFIGS
    from paper_1909_07309_b200.inputs import uniform_pm1
    from paper_1909_07309_b200.problems import identity_pieces

    cfg = CONFIGS[cfg_name]
    pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    x = torch.from_numpy(uniform_pm1(A.n_dof, cfg.seed)).cuda()
    y = A.apply(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        A.apply(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    np.save(out_path, y.cpu().numpy())
    return ms, A.n_dof


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        ms, n = run(sys.argv[2], sys.argv[3])
        print(f"{ms} {n}")
        sys.exit(0)
    import numpy as np

    for c in sys.argv[1:]:
        res = {}
        for mode in ("fused", "passes"):
            env = dict(os.environ)
            if mode == "passes":
                env["STIGA_MATVEC_PASSES"] = "1"
            path = f"/tmp/mv_{c}_{mode}.npy"
            out = subprocess.run([sys.executable, __file__, "--child", c, path], env=env, capture_output=True, text=True)
            if out.returncode != 0:
                print(c, mode, "FAILED", out.stderr[-1500:])
                break
            ms, n = out.stdout.split()
            res[mode] = (float(ms), int(n), path)
        if len(res) == 2:
            a, b = np.load(res["fused"][2]), np.load(res["passes"][2])
            rel = np.linalg.norm(a - b) / np.linalg.norm(b)
            n = res["fused"][1]
            print(f"{c}: N={n} fused {res['fused'][0]:.3f} ms ({48 * n / res['fused'][0] / 1e6:.0f} GB/s at 48 B/DoF)  "
                  f"passes {res['passes'][0]:.3f} ms  rel diff {rel:.2e}", flush=True)
