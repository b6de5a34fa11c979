"""Device stages of the time-sharded apply (stiga_fd_apply_space / _time / stiga_copy_blocks) driven
for W virtual ranks inside ONE process on one GPU: every rank's stages run with its real slab
offsets (t0, s0 > 0) and the all-to-all is replaced by the equivalent block copies between the
ranks' buffers (no kernel waits on another rank)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fdsolve as ofd  # noqa: E402
from paper_1909_07309_b200 import stiga  # noqa: E402
from paper_1909_07309_b200.distributed import DeviceBackend, ShardedExtendedFD  # noqa: E402
from paper_1909_07309_b200.inputs import uniform_pm1  # noqa: E402
from paper_1909_07309_b200.problems import identity_pieces  # noqa: E402

pytestmark = pytest.mark.gpu


def virtual_sharded_apply(P, r, world):
    ranks = [ShardedExtendedFD(DeviceBackend(P), P.dims, world=world, rank=q) for q in range(world)]
    sends = []
    for sh in ranks:
        a, b = sh.plan.local_slice()
        sends.append(sh.stage_forward(r[a:b].clone()))
    # forward all-to-all: rank q receives from r the block of size s_len[q]*t_len[r], in rank order
    for q, shq in enumerate(ranks):
        z = shq._bufs[2]
        off_out = 0
        for rr, shr in enumerate(ranks):
            off_in = sum(shr.plan.send_splits_fwd()[:q])
            n = shr.plan.send_splits_fwd()[q]
            z[off_out:off_out + n].copy_(sends[rr][off_in:off_in + n])
            off_out += n
    for sh in ranks:
        sh.stage_time()
    # backward all-to-all into each rank's `send` buffer
    for rr, shr in enumerate(ranks):
        recv = shr._bufs[1]
        off_out = 0
        for q, shq in enumerate(ranks):
            z2 = shq._bufs[3]
            off_in = sum(shq.plan.recv_splits_fwd()[:rr])
            n = shq.plan.recv_splits_fwd()[rr]
            recv[off_out:off_out + n].copy_(z2[off_in:off_in + n])
            off_out += n
    outs = [sh.stage_backward(torch.empty(sh.plan.local_size, dtype=torch.float64, device="cuda")) for sh in ranks]
    return torch.cat(outs)


@pytest.mark.parametrize("variant", ["fused", "split"])
@pytest.mark.parametrize("world,d,p,nel", [(1, 2, 3, 9), (2, 2, 3, 9), (3, 3, 2, 6), (4, 2, 2, 30), (8, 3, 3, 12)])
def test_virtual_ranks_match_oracle(variant, world, d, p, nel, monkeypatch):
    monkeypatch.setenv("STIGA_TIME_VARIANT", variant)
    pc = identity_pieces(d, p, nel)
    D = np.exp(0.3 * uniform_pm1(pc.n_dof, 3))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(pc.n_dof, 4)
    s = virtual_sharded_apply(P, torch.from_numpy(r).cuda(), world).cpu().numpy()
    so = Po.apply(r)
    assert np.linalg.norm(s - so) / np.linalg.norm(so) <= 1e-11


def virtual_sharded_matvec(A, x, world):
    """ShardedSystem stages for `world` virtual ranks; the halo exchange becomes block copies."""
    from paper_1909_07309_b200.distributed import DeviceSystemBackend, ShardedSystem

    ranks = [ShardedSystem(DeviceSystemBackend(A), A.dims, world=world, rank=q) for q in range(world)]
    for sh in ranks:
        a, b = sh.plan.local_slice()
        sh.stage_space(x[a:b].clone())
    views = [sh.halo_views() for sh in ranks]
    for q in range(world):
        for m in range(2):  # a, b
            if q > 0:
                views[q][m]["recv_lo"].copy_(views[q - 1][m]["send_hi"])
            if q < world - 1:
                views[q][m]["recv_hi"].copy_(views[q + 1][m]["send_lo"])
    outs = [sh.stage_time(torch.empty(sh.plan.local_size, dtype=torch.float64, device="cuda")) for sh in ranks]
    return torch.cat(outs)


@pytest.mark.parametrize("world,d,p,nel", [(1, 2, 3, 9), (2, 2, 3, 9), (3, 3, 2, 6), (4, 1, 4, 30), (5, 2, 2, 14)])
def test_virtual_ranks_spacetime_matvec(world, d, p, nel):
    pc = identity_pieces(d, p, nel)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.3, 0.7)
    x = torch.from_numpy(uniform_pm1(pc.n_dof, 6)).cuda()
    y = virtual_sharded_matvec(A, x, world)
    yo = A.apply(x)
    assert torch.linalg.norm(y - yo) <= 1e-13 * torch.linalg.norm(yo)


@pytest.mark.parametrize("pid,p,nel,world", [("deformed-cube-3d", 2, 3, 2), ("quarter-annulus-2d", 3, 8, 3)])
def test_virtual_ranks_physical_matvec(pid, p, nel, world):
    from paper_1909_07309_b200.problems import Problem

    A = stiga.KronSumOperator.physical(Problem(pid), p, nel)
    x = torch.from_numpy(uniform_pm1(A.n_dof, 7)).cuda()
    y = virtual_sharded_matvec(A, x, world)
    yo = A.apply(x)
    assert torch.linalg.norm(y - yo) <= 1e-13 * torch.linalg.norm(yo)


def test_sharded_gmres_driver_on_device_matches_native():
    """sharded_gmres (Python driver, device BLAS-1 through the C ABI) at world 1 vs the native
    stiga_gmres: same iteration count and solution."""
    from paper_1909_07309_b200.distributed import DeviceSystemBackend, DeviceVec, ShardedSystem, sharded_gmres

    pc = identity_pieces(2, 3, 10)
    D = np.exp(0.4 * uniform_pm1(pc.n_dof, 3))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    b = torch.from_numpy(uniform_pm1(pc.n_dof, 8)).cuda()
    Ash = ShardedSystem(DeviceSystemBackend(A), A.dims, world=1, rank=0)
    Psh = ShardedExtendedFD(DeviceBackend(P), P.dims, world=1, rank=0)
    x, rep = sharded_gmres(Ash, Psh, b, DeviceVec(), 1e-8, 200, 7)
    xn, repn = stiga.gmres(A, P, b, stiga.GmresOptions(1e-8, 200, 7))
    assert rep.converged and repn.converged and rep.iterations > 3
    assert abs(rep.iterations - repn.iterations) <= 1
    assert torch.linalg.norm(x - xn) <= 1e-8 * torch.linalg.norm(xn)


def test_slab_stage_argument_errors():
    """The slab stages reject what the reference's operators would reject (invalid_argument ->
    ValueError): generic-term operators, halo widths other than min(p, slices that exist), slabs
    outside [0, n_t), aliasing outputs."""
    import ctypes

    from paper_1909_07309_b200._lib import check, lib
    from paper_1909_07309_b200.distributed import DeviceSystemBackend

    pc = identity_pieces(2, 2, 6)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    be = DeviceSystemBackend(A)
    p = be.halfband()
    ns, nt = int(np.prod(A.dims[:-1])), A.dims[-1]
    x = torch.zeros(ns * nt, dtype=torch.float64, device="cuda")
    a, b, y = torch.zeros_like(x), torch.zeros_like(x), torch.zeros_like(x)
    with pytest.raises(ValueError):
        be.time(a, b, y, 2, 2, p + 1, p)  # wrong lower halo
    with pytest.raises(ValueError):
        be.time(a, b, y, nt - 1, 2, p, 0)  # slab past n_t
    with pytest.raises(ValueError):
        be.time(a, b, a, 0, 2, 0, p)  # output aliases an input
    with pytest.raises(ValueError):
        be.space(x, x, b, nt)  # output aliases the input
    G = stiga.KronSumOperator(A.dims, [(1.0, [np.eye(n) for n in A.dims])])
    with pytest.raises(ValueError):
        DeviceSystemBackend(G).halfband()
    r = torch.ones(10, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    check(lib().stiga_vec_dot(ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(r.data_ptr()), 10,
                              ctypes.c_void_p(out.data_ptr()), None), "vec_dot")
    assert out.item() == 10.0
    with pytest.raises(ValueError):
        check(lib().stiga_vec_dot(None, None, 10, ctypes.c_void_p(out.data_ptr()), None), "vec_dot")


# ---- fused exchange (scatter epilogues over peer memory) ---------------------------------------


def virtual_fused_apply(P, r, world):
    """FusedShardedExtendedFD for `world` virtual ranks on one GPU: the receive buffers are ordinary
    local tensors, so the scatter epilogues write into the other virtual ranks' buffers exactly as
    they would write into peer memory; stages run rank after rank (nothing waits on another rank)."""
    from paper_1909_07309_b200.distributed import FusedShardedExtendedFD, ShardPlan

    plans = [ShardPlan.make(P.dims, world, q) for q in range(world)]
    pl0 = plans[0]
    slab = [torch.full((pl0.s_len[q] * pl0.n_t,), float("nan"), dtype=torch.float64, device="cuda")
            for q in range(world)]
    tsl = [torch.full((pl0.n_s * pl0.t_len[q],), float("nan"), dtype=torch.float64, device="cuda")
           for q in range(world)]
    ranks = [FusedShardedExtendedFD(P, P.dims, q, world, [t.data_ptr() for t in slab], [t.data_ptr() for t in tsl])
             for q in range(world)]
    for f in ranks:
        a, b = f.plan.local_slice()
        f.stage_forward(r[a:b].clone())
    assert not any(torch.isnan(t).any() for t in slab), "forward scatter left a hole"
    for f in ranks:
        f.stage_time()
    assert not any(torch.isnan(t).any() for t in tsl), "time scatter left a hole"
    outs = [f.stage_backward(torch.empty(f.plan.local_size, dtype=torch.float64, device="cuda")) for f in ranks]
    return torch.cat(outs)


@pytest.mark.parametrize("fold", ["off", "auto", "force_wm2"])
@pytest.mark.parametrize("variant", ["fused", "split"])
@pytest.mark.parametrize("world,d,p,nel", [(1, 2, 3, 9), (2, 2, 3, 9), (3, 3, 2, 6), (4, 1, 4, 30), (8, 3, 3, 12),
                                           (5, 2, 2, 40)])
def test_virtual_ranks_fused_exchange(fold, variant, world, d, p, nel, monkeypatch):
    """Scatter-epilogue path = oracle (<= 1e-11); with dense kernels bit-identical to the pack +
    all-to-all path.  fold = force_wm2 restricts every split direction to folded WM = 2 tilings, so
    the last forward product runs the folded kernel's own scatter epilogue (fold_kernels.cu); with
    folded kernels the two paths agree to rounding."""
    monkeypatch.setenv("STIGA_TIME_VARIANT", variant)
    if fold != "auto":
        monkeypatch.setenv("STIGA_FOLD_KERNEL", fold)
    pc = identity_pieces(d, p, nel)
    D = np.exp(0.3 * uniform_pm1(pc.n_dof, 3))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
    Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
    r = uniform_pm1(pc.n_dof, 4)
    rt = torch.from_numpy(r).cuda()
    if fold == "force_wm2" and P.dims[0] >= 2 and d > 1:  # (d = 1: the scatter product cannot also pre-scale)
        names = [nm for nm, _ in P.launch_info()]
        assert any(nm.startswith(f"fwd_mode{d - 1}(folded)") for nm in names), names  # folded scatter epilogue
    s = virtual_fused_apply(P, rt, world)
    so = Po.apply(r)
    assert np.linalg.norm(s.cpu().numpy() - so) / np.linalg.norm(so) <= 1e-11
    sr = virtual_sharded_apply(P, rt, world)
    if fold == "off":
        assert torch.equal(s, sr)
    else:
        assert torch.linalg.norm(s - sr) <= 1e-13 * torch.linalg.norm(sr)


def test_scatter_stage_argument_errors():
    import ctypes

    from paper_1909_07309_b200._lib import check, lib
    from paper_1909_07309_b200.distributed import ShardPlan, scatter_desc, scatter_fields

    pc = identity_pieces(2, 2, 6)
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=0)
    pl = ShardPlan.make(P.dims, 2, 0)
    x = torch.zeros(P.n_dof, dtype=torch.float64, device="cuda")
    good = scatter_fields(pl, "space", [x.data_ptr(), x.data_ptr()])
    L = lib()

    def space(f, t0=0, ntl=pl.t_len[0]):
        check(L.stiga_fd_apply_space_scatter(P.handle, t0, ntl, ctypes.c_void_p(x.data_ptr()),
                                             ctypes.byref(scatter_desc(f)), None), "scatter")

    with pytest.raises(ValueError):  # time-stage descriptor on the space stage
        space(scatter_fields(pl, "time", [x.data_ptr(), x.data_ptr()]))
    with pytest.raises(ValueError):  # offsets do not cover N_s
        space(dict(good, offsets=[0, 3, 5]))
    with pytest.raises(ValueError):  # null destination
        space(dict(good, dst=[x.data_ptr(), None]))
    with pytest.raises(ValueError):  # slab outside [0, n_t)
        space(good, t0=pl.n_t - 1, ntl=2)


def _ipc_worker(rank, world, port, q):
    """One process per (virtual) rank, all on cuda:0: receive buffers exported with CUDA IPC and
    opened by the peer process; gloo host barriers (kernels never wait on another process)."""
    import os

    import torch.distributed as dist

    from paper_1909_07309_b200.distributed import FusedShardedExtendedFD

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pc = identity_pieces(2, 3, 11)
        D = np.exp(0.3 * uniform_pm1(pc.n_dof, 3))
        P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
        r = uniform_pm1(pc.n_dof, 4)
        f = FusedShardedExtendedFD.create(P, P.dims, device=0)
        a, b = f.plan.local_slice()
        x = torch.from_numpy(r[a:b].copy()).cuda()
        out = f.apply(x)
        out = f.apply(x)  # second apply reuses the exchanged buffers
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, out.cpu().numpy())
        dist.barrier()
        f.close()
        if rank == 0:
            Po = ofd.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D)
            so = Po.apply(r)
            s = np.concatenate(parts)
            q.put(float(np.linalg.norm(s - so) / np.linalg.norm(so)))
    finally:
        dist.destroy_process_group()


def test_fused_exchange_two_processes_cuda_ipc():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    assert q.get(timeout=5) <= 1e-11


def test_device_batched_gram_schmidt_ops():
    """stiga_vec_multidot / stiga_vec_multiaxpy (the CGS2 building blocks) against torch, k up to 130:
    cycles longer than the kernels' 64-vector limit are chunked inside DeviceVec."""
    from paper_1909_07309_b200.distributed import DeviceVec

    n = 100_003
    g = torch.Generator(device="cuda").manual_seed(3)
    V = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5 for _ in range(130)]
    w = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    vec = DeviceVec()
    for k in (1, 7, 8, 9, 20, 64, 65, 130):
        h = vec.multidot(V[:k], w)
        ref = np.array([float(torch.dot(v, w)) for v in V[:k]])
        assert np.abs(h - ref).max() <= 1e-12 * np.abs(ref).max()
        c = np.linspace(-1.0, 1.0, k)
        w2 = w.clone()
        vec.multiaxpy(c, V[:k], w2)
        ref2 = w + sum(float(c[j]) * V[j] for j in range(k))
        assert torch.linalg.norm(w2 - ref2) <= 1e-13 * torch.linalg.norm(ref2)


def test_sharded_gmres_cgs2_on_device_matches_native():
    """sharded_gmres with batched CGS2 orthogonalisation (two all-reduces per Arnoldi column) vs the
    native MGS stiga_gmres: iterations within one, same solution."""
    from paper_1909_07309_b200.distributed import DeviceSystemBackend, DeviceVec, ShardedSystem, sharded_gmres

    pc = identity_pieces(2, 3, 10)
    D = np.exp(0.4 * uniform_pm1(pc.n_dof, 3))
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=0)
    A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0)
    b = torch.from_numpy(uniform_pm1(pc.n_dof, 8)).cuda()
    Ash = ShardedSystem(DeviceSystemBackend(A), A.dims, world=1, rank=0)
    Psh = ShardedExtendedFD(DeviceBackend(P), P.dims, world=1, rank=0)
    x, rep = sharded_gmres(Ash, Psh, b, DeviceVec(), 1e-8, 200, 7, ortho="cgs2")
    xn, repn = stiga.gmres(A, P, b, stiga.GmresOptions(1e-8, 200, 7))
    assert rep.converged and repn.converged and rep.iterations > 3
    assert abs(rep.iterations - repn.iterations) <= 1
    assert torch.linalg.norm(x - xn) <= 1e-8 * torch.linalg.norm(xn)


def test_bench_two_ranks_share_one_gpu_gloo():
    """bench.py's N > 1 path end to end with two ranks on this one GPU (STIGA_BENCH_BACKEND=gloo):
    receive buffers exchanged with CUDA IPC, the time-sharded apply with the fused scatter exchange,
    the halo-exchanged system mat-vec and the CGS2 sharded GMRES; one JSON line, converged solve."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, STIGA_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    # no launcher: bench.py --gpus 2 starts its two ranks itself (torch.distributed.run on 127.0.0.1)
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "5",
           "--warmup", "3"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "scatter epilogues" in d["config"]["parallelism"]
    assert any(k.startswith("exchange_barrier") for k in d["pass_ms"])
    assert d["gmres"]["converged"] and d["gmres"]["true_rel_residual"] < 1e-8
