"""Debugging aid: accuracy of the GPU FD apply and of the float64 oracle against an extended-
precision (x87 long double) evaluation of the same apply on the product's exported factors, for a
d = 1 shape (usage: python tools/precision_probe.py p n_el [scaled])."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from oracle import fdsolve as ofd  # noqa: E402
from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import identity_pieces  # noqa: E402
from test_fd_gpu import _oracle_with_product_basis  # noqa: E402

LD = np.longdouble
p, nel = int(sys.argv[1]), int(sys.argv[2])
scaled = len(sys.argv) > 3
pc = identity_pieces(1, p, nel)
nd = pc.K[0].shape[0] * pc.Wt.shape[0]
D = np.exp(0.3 * uniform_pm1(nd, 32)) if scaled else None
r = uniform_pm1(nd, 31)
P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
s_gpu = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
Pb = _oracle_with_product_basis(ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D),
                                P, 1)
s_or = Pb.apply(r)
Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
s_o = Po.apply(r)


def ld_apply(Pb, r):
    lu = Pb.lu
    U, Ut = Pb.U[0].astype(LD), Pb.time.U.astype(LD)
    ns, nt = U.shape[0], Ut.shape[0]
    x = r.astype(LD)
    if Pb.d_inv_sqrt is not None:
        x = Pb.d_inv_sqrt.astype(LD) * x
    X = x.reshape(nt, ns).T                      # X[i, t]
    Z = (U.T @ X) @ Ut                           # U_s^T X U_t  (time mode: x_b . J^T with J = U_t^T)
    lam = lu.lambda_s.astype(LD)
    li = 1 / lam
    g = np.asarray(lu.g, dtype=LD)
    gam, nu = LD(lu.gamma), LD(lu.nu)
    S = Z.T.copy()                               # rows = time eigen-coordinates
    Xo = np.empty_like(S)
    srhs = S[nt - 1].copy()
    Rinv = []
    for j, lt in enumerate(lu.lambda_t):
        lt = LD(lt)
        c = gam * gam / nu * lt * lt
        R = 1 / (nu * lam + c * li)
        Rinv.append(R)
        c1 = gam / nu * lt
        u, w = S[2 * j], S[2 * j + 1]
        xa = li * u / nu - (c1 * c1 / nu) * (li * (R * (li * u))) - c1 * (li * (R * w))
        xb = c1 * (R * (li * u)) + R * w
        Xo[2 * j], Xo[2 * j + 1] = xa, xb
        srhs += gam * (g[2 * j] * xa + g[2 * j + 1] * xb)
    if lu.zero_count:
        z = nt - 2
        Xo[z] = li * S[z] / nu
        srhs += gam * g[z] * Xo[z]
    xl = lu.S_inv.astype(LD) * srhs
    Xo[nt - 1] = xl
    for j, lt in enumerate(lu.lambda_t):
        lt = LD(lt)
        c1 = gam / nu * lt
        R = Rinv[j]
        u, w = gam * g[2 * j] * xl, gam * g[2 * j + 1] * xl
        xa = li * u / nu - (c1 * c1 / nu) * (li * (R * (li * u))) - c1 * (li * (R * w))
        xb = c1 * (R * (li * u)) + R * w
        Xo[2 * j] -= xa
        Xo[2 * j + 1] -= xb
    if lu.zero_count:
        z = nt - 2
        Xo[z] -= li * (gam * g[z] * xl) / nu
    Y = (U @ Xo.T) @ Ut.T
    y = Y.T.reshape(-1)
    if Pb.d_inv_sqrt is not None:
        y = Pb.d_inv_sqrt.astype(LD) * y
    return y


s_ld = ld_apply(Pb, r)
nrm = float(np.linalg.norm(s_ld.astype(np.float64)))
err = lambda s: float(np.linalg.norm((s.astype(LD) - s_ld).astype(np.float64))) / nrm  # noqa: E731
print(f"p={p} n_el={nel} scaled={scaled}: |gpu - ld| {err(s_gpu):.3e}  |oracle(product basis) - ld| {err(s_or):.3e}  "
      f"|oracle(own basis) - ld| {err(s_o):.3e}  |gpu - oracle| {np.linalg.norm(s_gpu - s_o) / np.linalg.norm(s_o):.3e}")

# ---- stage-by-stage: each device stage fed the (rounded) long-double input of that stage -------
import ctypes  # noqa: E402

from paper_1909_07309_b200._lib import check, lib  # noqa: E402

ns, nt = Pb.U[0].shape[0], Pb.time.U.shape[0]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def stage_space(x, backward):
    out = torch.empty_like(x)
    check(lib().stiga_fd_apply_space(P.handle, int(backward), 0, nt, ctypes.c_void_p(x.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()), None), "space")
    torch.cuda.synchronize()
    return out.cpu().numpy()


def stage_time(z):
    # time stage wants the spatial-slab layout (ns_local x n_t colex) == the full vector for one slab
    out = torch.empty_like(z)
    check(lib().stiga_fd_apply_time(P.handle, 0, ns, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                    None), "time")
    torch.cuda.synchronize()
    return out.cpu().numpy()


# device order of the spatial eigen-index: [symmetric eigenvectors; skew ones] when split (d = 1)
import copy  # noqa: E402

Ua = Pb.U[0]
split = os.environ.get("STIGA_NO_FOLD") is None
symm = Ua[0] * Ua[-1] > 0
order = np.concatenate([np.nonzero(symm)[0], np.nonzero(~symm)[0]]) if split else np.arange(ns)
Ud = Ua[:, order]
scl = Pb.d_inv_sqrt.astype(LD) if Pb.d_inv_sqrt is not None else np.ones(nd, dtype=LD)
Z1 = Ud.astype(LD).T @ (r.astype(LD) * scl).reshape(nt, ns).T      # (ns, nt), device eigen order
z1 = stage_space(dev(r), False).reshape(nt, ns).T


def rel(a, b):
    return float(np.linalg.norm((a.astype(LD) - b).astype(np.float64)) / np.linalg.norm(b.astype(np.float64)))


print("forward space stage:", rel(z1, Z1))
Zr = Z1.astype(np.float64)
Pt = copy.deepcopy(Pb)
lu = Pt.lu
lu.lambda_s, lu.lambda_s_inv, lu.S_inv = lu.lambda_s[order], lu.lambda_s_inv[order], lu.S_inv[order]
lu.R_inv = [q[order] for q in lu.R_inv]
Pt.U = [np.eye(ns)]
Pt.d_inv_sqrt = None
vin = Zr.T.reshape(-1)
t_ld = ld_apply(Pt, vin)
t_gpu = stage_time(dev(vin))
print("time stage:", rel(t_gpu, t_ld))
# float64 oracle on the same time stage
Pt64 = copy.deepcopy(Pt)
Pt64.transform = [np.eye(ns), Pt.time.U]
Pt64.transform_t = [np.eye(ns), Pt.time.U.T.copy()]
print("time stage oracle f64:", rel(Pt64.apply(vin), t_ld))
E = np.abs((t_gpu.astype(LD) - t_ld).astype(np.float64)).reshape(nt, ns)
Tn = np.abs(t_ld.astype(np.float64)).reshape(nt, ns)
per_s = E.max(axis=0) / max(Tn.max(), 1e-300)
top = np.argsort(per_s)[::-1][:8]
print("worst spatial indices (device order):", top, "lambda_s:", lu.lambda_s[top], "err/max:", per_s[top])
per_t = E.max(axis=1) / Tn.max()
print("worst time rows:", np.argsort(per_t)[::-1][:8], per_t[np.argsort(per_t)[::-1][:8]])
print("output magnitude by time row (max):", Tn.max(axis=1)[:4], Tn.max(axis=1)[-4:])
if os.environ.get("STIGA_DEBUG_ARROW") == "1":   # fused time kernel without the arrowhead: X U_t U_t^T
    Xv = vin.astype(LD).reshape(nt, ns).T
    Ut = Pb.time.U.astype(LD)
    g_ld = ((Xv @ Ut) @ Ut.T).T.reshape(-1)
    print("time GEMMs only (U_t U_t^T):", rel(t_gpu, g_ld))
    Zg = (Xv @ Ut)
    print("  |U_t^T x| column-0 magnitude:", float(np.abs(Zg[0].astype(np.float64)).max()), "max:",
          float(np.abs(Zg.astype(np.float64)).max()))
# arrowhead output of the device for the worst column, recovered by undoing the final U_t product
c0 = int(np.argmin(lu.lambda_s))
Ut64 = Pb.time.U
Tg = t_gpu.reshape(nt, ns)[:, c0]            # = U_t @ xo  (time mode, J = U_t)
Tl = t_ld.reshape(nt, ns)[:, c0].astype(np.float64)
xo_g = np.linalg.solve(Ut64, Tg)
xo_l = np.linalg.solve(Ut64, Tl)
d = np.abs(xo_g - xo_l)
print("arrowhead rows of the worst column: x_last gpu/ld", xo_g[-1], xo_l[-1], "rel", abs(xo_g[-1] - xo_l[-1]) / abs(xo_l[-1]))
print("  zero row", xo_g[-2], xo_l[-2], " worst rows", np.argsort(d)[::-1][:6], (d / np.abs(xo_l).max())[np.argsort(d)[::-1][:6]])
# device Z = (I (x) U_t^T) x through stiga_kron_matvec (same DMMA mode kernel) vs long double
Zd = stiga.kron_matvec([np.eye(ns), Ut64.T], dev(vin)).cpu().numpy().reshape(nt, ns)
Zl = (vin.astype(LD).reshape(nt, ns).T @ Ut64.astype(LD)).T       # (nt, ns)
dz = np.abs((Zd.astype(LD) - Zl).astype(np.float64))
print("Z via kron_matvec: worst column-0 rows", np.argsort(dz[:, c0])[::-1][:4],
      (dz[:, c0] / np.abs(Zl[:, c0].astype(np.float64)))[np.argsort(dz[:, c0])[::-1][:4]],
      "global rel", float(np.linalg.norm(dz) / np.linalg.norm(Zl.astype(np.float64))))
print("x_last gpu / ld:", xo_g[-1], xo_l[-1])
# same long-double reference, but with the product's own eigenvalues Lambda_s (ascending export)
lam_p = P.export(1, 0)
print("lambda_min product / oracle:", lam_p[0], Pb.lu.lambda_s[0], "rel", abs(lam_p[0] - Pb.lu.lambda_s[0]) / lam_p[0])
Pc = copy.deepcopy(Pb)
Pc.lu.lambda_s = lam_p.copy()
Pc.lu.lambda_s_inv = 1.0 / lam_p
s_ldp = ld_apply(Pc, r)
print("gpu vs long double on the product's Lambda_s:",
      float(np.linalg.norm((s_gpu.astype(LD) - s_ldp).astype(np.float64)) / np.linalg.norm(s_ldp.astype(np.float64))))
