"""Time-sharded FD apply (paper_1909_07309_b200/distributed.py) with world_size 2 and 3 over gloo on
CPU.  The stage compute is the oracle (oracle/) so the test exercises the product's partition,
pack/unpack and all-to-all logic; the GPU stages are the same C ABI calls tested in test_fd_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fdsolve as ofd
from oracle.kronop import mode_product
from paper_1909_07309_b200.distributed import ShardedExtendedFD, ShardPlan, partition


class OracleBackend:
    """CPU stand-in for the device stages, built from the oracle's pieces."""

    def __init__(self, Po):
        self.Po = Po
        self.d = len(Po.U)
        self.dims = Po.dims

    def space(self, x, out, backward, t0, ntl):
        P = self.Po
        n_s = int(np.prod(self.dims[:-1]))
        v = x.numpy().copy()
        dims = list(self.dims[:-1]) + [ntl]
        dsl = None if P.d_inv_sqrt is None else P.d_inv_sqrt[n_s * t0:n_s * (t0 + ntl)]
        if not backward and dsl is not None:
            v = dsl * v
        for m in range(self.d):
            v, dims = mode_product(v, dims, P.U[m] if backward else P.U[m].T, m)
        if backward and dsl is not None:
            v = dsl * v
        out.copy_(torch.from_numpy(v))

    def time(self, z, out, s0, nsl):
        P = self.Po
        nt = self.dims[-1]
        v, dims = mode_product(z.numpy(), [nsl, nt], P.time.U.T, 1)
        lu = ofd.ArrowheadLU()
        full = P.lu
        lu.gamma, lu.nu = full.gamma, full.nu
        lu.lambda_s = full.lambda_s[s0:s0 + nsl]
        lu.lambda_s_inv = full.lambda_s_inv[s0:s0 + nsl]
        lu.lambda_t, lu.zero_count, lu.g, lu.sigma = full.lambda_t, full.zero_count, full.g, full.sigma
        lu.R_inv = [r[s0:s0 + nsl] for r in full.R_inv]
        lu.S_inv = full.S_inv[s0:s0 + nsl]
        v = ofd.arrowhead_solve(lu, v)
        v, _ = mode_product(v, dims, P.time.U, 1)
        out.copy_(torch.from_numpy(v))

    def copy_blocks(self, src, src_off, sld, dst, dst_off, dld, rows, cols):
        for r in range(rows):
            dst[dst_off + r * dld: dst_off + r * dld + cols] = src[src_off + r * sld: src_off + r * sld + cols]


def _problem(d, p, nel, scaled):
    from oracle.assembly import assemble_spatial_parametric, assemble_time_matrices

    W, Mt = assemble_time_matrices(p, nel, 1.0)
    K, M = assemble_spatial_parametric(p, nel, d)
    n = K[0].shape[0] ** d * W.shape[0]
    D = np.random.default_rng(5).uniform(0.5, 2.0, n) if scaled else None
    return ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=D)


def _worker(rank, world, port, d, p, nel, scaled, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Po = _problem(d, p, nel, scaled)
        r = np.random.default_rng(9).uniform(-1, 1, Po.n_dof)
        sh = ShardedExtendedFD(OracleBackend(Po), Po.dims)
        a, b = sh.plan.local_slice()
        out = sh.apply(torch.from_numpy(r[a:b].copy()))
        parts = [None] * world
        dist.all_gather_object(parts, out.numpy())
        if rank == 0:
            s = np.concatenate(parts)
            so = Po.apply(r)
            q.put(float(np.linalg.norm(s - so) / np.linalg.norm(so)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,d,p,nel,scaled", [(2, 2, 2, 6, True), (3, 2, 3, 5, False), (2, 3, 2, 3, True),
                                                   (2, 1, 3, 9, True)])
def test_sharded_apply_matches_oracle(world, d, p, nel, scaled):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, p, nel, scaled, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    assert q.get(timeout=5) <= 1e-12


def test_partition_and_plan():
    assert partition(10, 3) == ([0, 4, 7], [4, 3, 3])
    pl = ShardPlan.make([5, 5, 7], 3, 1)
    assert pl.n_s == 25 and pl.t_len == [3, 2, 2] and pl.s_len == [9, 8, 8]
    assert pl.local_slice() == (75, 125)
    assert sum(pl.send_splits_fwd()) == pl.local_size
    assert sum(pl.recv_splits_fwd()) == pl.s_len[1] * pl.n_t
    with pytest.raises(ValueError):
        ShardPlan.make([3, 2], 3, 0)


def test_single_rank_degenerates():
    Po = _problem(2, 2, 4, True)
    r = np.random.default_rng(2).uniform(-1, 1, Po.n_dof)
    sh = ShardedExtendedFD(OracleBackend(Po), Po.dims)
    s = sh.apply(torch.from_numpy(r.copy())).numpy()
    assert np.linalg.norm(s - Po.apply(r)) <= 1e-12 * np.linalg.norm(s)


# ---- fused exchange: scatter descriptors (host logic of FusedShardedExtendedFD) ----------------


def scatter_model(fields, values, A, bufs):
    """numpy restatement of the kernel scatter epilogue (fd_kernels.cu store_acc_scatter) driven by
    the same descriptor fields: element e of a stage output (a = e mod A, b = e div A) is stored into
    bufs[q], q the owner of a (space stage) or b (time stage)."""
    e = np.arange(values.size)
    a, b = e % A, e // A
    bt = fields["by_time"]
    off = np.asarray(fields["offsets"])
    key = b if bt else a
    q = np.searchsorted(off, key, side="right") - 1
    for k in range(fields["world"]):
        sel = q == k
        da = a[sel] - (0 if bt else off[k]) + fields["a_shift"]
        db = b[sel] - (off[k] if bt else 0) + fields["b_shift"]
        bufs[k][da + fields["ld"][k] * db] = values[sel]


@pytest.mark.parametrize("world,d,p,nel,scaled", [(2, 2, 2, 6, True), (3, 2, 3, 5, False), (3, 3, 2, 3, True),
                                                   (8, 2, 2, 9, True), (2, 1, 3, 9, True)])
def test_fused_exchange_descriptors_match_oracle(world, d, p, nel, scaled):
    """Virtual ranks: forward stage -> scatter into the owners' slab buffers -> time stage -> scatter
    into the owners' time-slab buffers -> backward stage equals the unsharded oracle apply, and every
    receive element is written exactly once."""
    from paper_1909_07309_b200.distributed import scatter_fields

    Po = _problem(d, p, nel, scaled)
    be = OracleBackend(Po)
    r = np.random.default_rng(9).uniform(-1, 1, Po.n_dof)
    plans = [ShardPlan.make(Po.dims, world, q) for q in range(world)]
    pl0 = plans[0]
    slab = [np.full(pl0.s_len[q] * pl0.n_t, np.nan) for q in range(world)]
    tslab = [np.full(pl0.n_s * pl0.t_len[q], np.nan) for q in range(world)]
    hits = [np.zeros(b.size, int) for b in slab]
    for pl in plans:
        a, b = pl.local_slice()
        y = torch.empty(pl.local_size, dtype=torch.float64)
        be.space(torch.from_numpy(r[a:b].copy()), y, False, pl.t_off[pl.rank], pl.t_len[pl.rank])
        f = scatter_fields(pl, "space", list(range(world)))
        scatter_model(f, y.numpy(), pl.n_s, slab)
        scatter_model(f, np.ones(y.numel()), pl.n_s, hits)
    assert all((h == 1).all() for h in hits)
    for pl in plans:
        z = torch.empty(pl.s_len[pl.rank] * pl.n_t, dtype=torch.float64)
        be.time(torch.from_numpy(slab[pl.rank]), z, pl.s_off[pl.rank], pl.s_len[pl.rank])
        scatter_model(scatter_fields(pl, "time", list(range(world))), z.numpy(), pl.s_len[pl.rank], tslab)
    assert not any(np.isnan(t).any() for t in tslab)
    outs = []
    for pl in plans:
        o = torch.empty(pl.local_size, dtype=torch.float64)
        be.space(torch.from_numpy(tslab[pl.rank]), o, True, pl.t_off[pl.rank], pl.t_len[pl.rank])
        outs.append(o.numpy())
    s, so = np.concatenate(outs), Po.apply(r)
    assert np.linalg.norm(s - so) <= 1e-12 * np.linalg.norm(so)


def test_scatter_desc_fields_and_limits():
    from paper_1909_07309_b200.distributed import scatter_desc, scatter_fields

    pl = ShardPlan.make([5, 5, 7], 3, 1)
    f = scatter_fields(pl, "space", [10, 20, 30])
    assert f["offsets"] == [0, 9, 17, 25] and f["ld"] == [9, 8, 8] and f["b_shift"] == 3 and f["by_time"] == 0
    g = scatter_fields(pl, "time", [10, 20, 30])
    assert g["offsets"] == [0, 3, 5, 7] and g["ld"] == [25] * 3 and g["a_shift"] == 9 and g["by_time"] == 1
    d = scatter_desc(g)
    assert d.world == 3 and list(d.offsets)[:4] == [0, 3, 5, 7] and d.dst[2] == 30
    with pytest.raises(ValueError):
        scatter_fields(pl, "space", [1, 2])
    with pytest.raises(ValueError):
        scatter_fields(pl, "bogus", [1, 2, 3])
    big = ShardPlan.make([40, 40, 12], 9, 0)
    with pytest.raises(ValueError):
        scatter_desc(scatter_fields(big, "space", list(range(9))))
