"""Time-sharded system mat-vec (halo exchange of the banded time factors) and the sharded GMRES
(all-reduced Krylov dots) of paper_1909_07309_b200/distributed.py, world_size 2 and 3 over gloo on
CPU.  Stage compute is the oracle; the product code under test is the partition, the halo and
all-to-all exchanges and the GMRES control flow (gmres.cpp:19-132 with distributed dots)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import assembly as oasm
from oracle import fdsolve as ofd
from oracle import gmres as ogm
from oracle import kronop as okr
from oracle.kronop import mode_product
from paper_1909_07309_b200.distributed import ShardedExtendedFD, ShardedSystem, sharded_gmres

from test_distributed import OracleBackend, _free_port


class OracleSystemBackend:
    """CPU stand-in for stiga_kronsum_apply_space / _apply_time of the spacetime form."""

    def __init__(self, K, M, Wt, Mt, gamma, nu):
        self.K, self.M = K, M
        self.Wt, self.Mt = gamma * np.asarray(Wt), nu * np.asarray(Mt)
        self.ns = [k.shape[0] for k in K]
        self.nt = self.Wt.shape[0]

    def halfband(self):
        def hb(F):
            i, j = np.nonzero(F)
            return int(np.max(np.abs(i - j))) if len(i) else 0

        return max(hb(self.Wt), hb(self.Mt))

    def space(self, x, a, b, ntl):
        d = len(self.K)
        dims = self.ns + [ntl]
        v = x.numpy()
        av, _ = mode_product(v, dims, self.M[0], 0)
        bv, _ = mode_product(v, dims, self.K[0], 0)
        for m in range(1, d):
            a2, _ = mode_product(av, dims, self.M[m], m)
            b2 = mode_product(av, dims, self.K[m], m)[0] + mode_product(bv, dims, self.M[m], m)[0]
            av, bv = a2, b2
        a.copy_(torch.from_numpy(av))
        b.copy_(torch.from_numpy(bv))

    def time(self, a_ext, b_ext, y, t0, ntl, hl, hh):
        ns = int(np.prod(self.ns))
        cols = slice(t0 - hl, t0 + ntl + hh)
        A2 = a_ext.numpy().reshape(-1, ns).T  # ns x (hl + ntl + hh)
        B2 = b_ext.numpy().reshape(-1, ns).T
        Y = A2 @ self.Wt[t0:t0 + ntl, cols].T + B2 @ self.Mt[t0:t0 + ntl, cols].T
        y.copy_(torch.from_numpy(Y.T.reshape(-1).copy()))


class CpuVec:
    def __init__(self, group=None):
        self.group = group

    def dot(self, x, y):
        s = torch.tensor([float(torch.dot(x, y))], dtype=torch.float64)
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(s)
        return float(s.item())

    def axpy(self, alpha, x, y):
        y.add_(x, alpha=alpha)

    def scal(self, alpha, x, y):
        torch.mul(x, alpha, out=y)

    def multidot(self, Vs, w):
        s = torch.tensor([float(torch.dot(v, w)) for v in Vs], dtype=torch.float64)
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(s)  # one collective for the whole column
        return s.numpy()

    def multiaxpy(self, coefs, Vs, w):
        for c, v in zip(coefs, Vs):
            w.add_(v, alpha=float(c))


def _setup(d, p, nel, gamma, nu, scaled):
    W, Mt = oasm.assemble_time_matrices(p, nel, 1.0)
    K, M = oasm.assemble_spatial_parametric(p, nel, d)
    dims = [K[0].shape[0]] * d + [W.shape[0]]
    n = int(np.prod(dims))
    D = np.exp(0.4 * np.random.default_rng(5).uniform(-1, 1, n)) if scaled else None
    Po = ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=D)
    Ao = okr.KronSumOperator(dims, oasm.kron_sum_terms(K, M, W, Mt, gamma, nu))
    return K, M, W, Mt, dims, Po, Ao


def _worker(rank, world, port, d, p, nel, gamma, nu, scaled, restart, q, ortho="mgs"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, M, W, Mt, dims, Po, Ao = _setup(d, p, nel, gamma, nu, scaled)
        Ash = ShardedSystem(OracleSystemBackend(K, M, W, Mt, gamma, nu), dims)
        Psh = ShardedExtendedFD(OracleBackend(Po), dims)
        a, b = Ash.plan.local_slice()
        rhs = np.random.default_rng(11).uniform(-1, 1, Ao.n_dof)
        # mat-vec parity
        y = Ash.apply(torch.from_numpy(rhs[a:b].copy()))
        parts = [None] * world
        dist.all_gather_object(parts, y.numpy())
        yerr = None
        if rank == 0:
            yo = Ao.apply(rhs)
            yerr = float(np.linalg.norm(np.concatenate(parts) - yo) / np.linalg.norm(yo))
        # GMRES parity
        x, rep = sharded_gmres(Ash, Psh, torch.from_numpy(rhs[a:b].copy()), CpuVec(), 1e-8, 200, restart, ortho=ortho)
        xs = [None] * world
        dist.all_gather_object(xs, x.numpy())
        if rank == 0:
            xo, repo = ogm.gmres(Ao.apply, Po.apply, rhs, 1e-8, 200, restart)
            xg = np.concatenate(xs)
            q.put((yerr, rep.iterations, repo.iterations, rep.converged,
                   float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,d,p,nel,gamma,nu,scaled,restart,ortho", [
    (2, 2, 2, 6, 1.0, 1.0, True, None, "mgs"),
    (3, 2, 3, 8, 1.3, 0.7, True, 5, "mgs"),
    (2, 1, 3, 12, 1.0, 1.0, True, 4, "mgs"),
    (3, 3, 2, 5, 1.0, 1.0, False, None, "mgs"),
    (2, 2, 2, 6, 1.0, 1.0, True, None, "cgs2"),
    (3, 2, 3, 8, 1.3, 0.7, True, 5, "cgs2"),
])
def test_sharded_system_and_gmres_match_oracle(world, d, p, nel, gamma, nu, scaled, restart, ortho):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, p, nel, gamma, nu, scaled, restart, q, ortho))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(240)
        assert pr.exitcode == 0
    yerr, its, its_o, conv, xerr = q.get(timeout=5)
    assert yerr <= 1e-13
    assert conv and abs(its - its_o) <= 1
    assert xerr <= 1e-6


def test_halo_needs_p_slices():
    class B:
        def halfband(self):
            return 3

    with pytest.raises(ValueError):
        ShardedSystem(B(), [4, 5], world=3, rank=0)  # slabs of 2/2/1 slices < p = 3
