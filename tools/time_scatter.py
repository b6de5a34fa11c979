"""Cost of the scatter epilogue (fused all-to-all) against the plain stores, per stage, for one rank
of a G-way time-sharded apply (virtual ranks on one GPU: the scatter targets are local buffers, so
this isolates the epilogue's index work from NVLink).  Usage: python tools/time_scatter.py c3 8"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench import problem_pieces  # noqa: E402
from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200._lib import check, lib  # noqa: E402
from paper_1909_07309_b200.configs import CONFIGS  # noqa: E402
from paper_1909_07309_b200.distributed import ShardPlan, scatter_desc, scatter_fields  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pc, D = problem_pieces(cfg, device=0)
P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
plans = [ShardPlan.make(P.dims, G, q) for q in range(G)]
pl = plans[0]
f64 = dict(dtype=torch.float64, device="cuda")
slab = [torch.empty(pl.s_len[q] * pl.n_t, **f64) for q in range(G)]
tsl = [torch.empty(pl.n_s * pl.t_len[q], **f64) for q in range(G)]
x = torch.rand(pl.local_size, **f64)
out = torch.empty_like(x)
z = torch.rand(pl.s_len[0] * pl.n_t, **f64)
zo = torch.empty_like(z)
fwd = scatter_desc(scatter_fields(pl, "space", [t.data_ptr() for t in slab]))
bwd = scatter_desc(scatter_fields(pl, "time", [t.data_ptr() for t in tsl]))
L = lib()
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def timed(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t0, ntl = pl.t_off[0], pl.t_len[0]
s0, nsl = pl.s_off[0], pl.s_len[0]
a = timed(lambda: check(L.stiga_fd_apply_space(P.handle, 0, t0, ntl, vp(x), vp(out), None), "space"))
b = timed(lambda: check(L.stiga_fd_apply_space_scatter(P.handle, t0, ntl, vp(x), ctypes.byref(fwd), None), "scatter"))
c = timed(lambda: check(L.stiga_fd_apply_time(P.handle, s0, nsl, vp(z), vp(zo), None), "time"))
d = timed(lambda: check(L.stiga_fd_apply_time_scatter(P.handle, s0, nsl, vp(z), ctypes.byref(bwd), None), "tscatter"))
print(f"{cfg.name} G={G} rank 0: forward spatial stage {a:.3f} ms plain / {b:.3f} ms scatter; "
      f"time stage {c:.3f} ms plain / {d:.3f} ms scatter")
