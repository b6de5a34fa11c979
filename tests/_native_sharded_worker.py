"""Worker of tests/test_native_sharded_gpu.py: one rank of the NATIVE time-sharded path (C ABI:
stiga_comm_init_host over a gloo process group, stiga_fd_setup_sharded, sharded KronSumOperator,
collective stiga_gmres), several ranks sharing one GPU.  Launched by torch.distributed.run; rank 0
checks the gathered results against the single-device product and the oracle and prints one JSON line.
Nothing waits on another rank inside a kernel: the host-callback communicator synchronizes the stream
before every barrier / reduction."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def gather(t):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, t.cpu().numpy())
    return np.concatenate(parts)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    case = sys.argv[1]
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    rank, world = dist.get_rank(), dist.get_world_size()
    from oracle import assembly as oasm
    from oracle import fdsolve as ofd
    from oracle import gmres as ogm
    from oracle import kronop as okr
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.inputs import uniform_pm1
    from paper_1909_07309_b200.problems import Problem, identity_pieces

    comm = stiga.Comm.from_process_group()
    out = {"case": case, "world": world}
    if case in ("spacetime", "memory"):
        d, p, nel = (2, 3, 9) if case == "spacetime" else (2, 3, 256)
        pc = identity_pieces(d, p, nel)
        K, M, Wt, Mt = pc.K, pc.M, pc.Wt, pc.Mt
        D = np.exp(0.3 * uniform_pm1(pc.n_dof, 3))
        A_single = None
    else:  # physical: curved geometry, A^G pieces with the geometry scaling
        prob = Problem("deformed-cube-3d")
        pc = prob.geometry_pieces(2, 6, want_D=True)
        K, M, Wt, Mt, D = pc.K, pc.M, pc.Wt, pc.Mt, pc.D
    n_dof = pc.n_dof
    n_s = n_dof // Wt.shape[0]
    t0, ntl = stiga.shard_partition(Wt.shape[0], world, rank)
    lo, hi = n_s * t0, n_s * (t0 + ntl)

    dist.barrier()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    dist.barrier()
    P = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D[lo:hi], comm=comm)
    torch.cuda.synchronize()
    dist.barrier()
    free1 = torch.cuda.mem_get_info()[0]
    out["fd_bytes_all_ranks"] = free0 - free1
    out["n_dof"] = n_dof
    assert P.local_slice() == (lo, hi)
    r = uniform_pm1(n_dof, 4)
    s_loc = P.apply(torch.from_numpy(r[lo:hi]).cuda())
    s = gather(s_loc)
    names = [nm for nm, _ in P.launch_info()]
    prof = P.apply_profiled(torch.from_numpy(r[lo:hi]).cuda(), torch.empty_like(s_loc))
    out["launches"] = names
    out["profiled_ok"] = len(prof) == len(names) and all(x >= 0 for x in prof)
    if case == "memory":
        del P
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            free2 = torch.cuda.mem_get_info()[0]
            P1 = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D, device=0)
            torch.cuda.synchronize()
            out["fd_bytes_single"] = free2 - torch.cuda.mem_get_info()[0]
            out["apply_vs_single"] = rel(s, P1.apply(torch.from_numpy(r).cuda()).cpu().numpy())
            print(json.dumps(out), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        return
    if rank == 0:
        Po = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D)
        out["apply_vs_oracle"] = rel(s, Po.apply(r))
        P1 = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 1.0, 1.0, scaling=D, device=0)
        out["apply_vs_single"] = rel(s, P1.apply(torch.from_numpy(r).cuda()).cpu().numpy())
    # system operator
    if case == "spacetime":
        A = stiga.KronSumOperator.spacetime(K, M, Wt, Mt, 1.0, 1.0, comm=comm)
        A1 = stiga.KronSumOperator.spacetime(K, M, Wt, Mt, 1.0, 1.0, device=0)
    else:
        A = stiga.KronSumOperator.physical(prob, 2, 6, comm=comm)
        A1 = stiga.KronSumOperator.physical(prob, 2, 6, device=0)
    x = uniform_pm1(n_dof, 5)
    y = gather(A.apply(torch.from_numpy(x[lo:hi]).cuda()))
    # repeated applies (halo buffers reused across calls)
    for _ in range(3):
        y2 = gather(A.apply(torch.from_numpy(x[lo:hi]).cuda()))
    y1 = A1.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    if rank == 0:
        out["matvec_vs_single"] = rel(y, y1)
        out["matvec_repeat_equal"] = bool(np.array_equal(y, y2))
        if case == "spacetime":
            Ao = okr.KronSumOperator(pc.dims, oasm.kron_sum_terms(K, M, Wt, Mt, 1.0, 1.0))
            out["matvec_vs_oracle"] = rel(y, Ao.apply(x))
    # collective GMRES (CGS2 over the communicator); a gamma-mismatched preconditioner makes it non-trivial
    b = uniform_pm1(n_dof, 6)
    Pg = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 0.4, 1.0, scaling=D[lo:hi], comm=comm)
    xs, rep = stiga.gmres(A, Pg, torch.from_numpy(b[lo:hi]).cuda(), stiga.GmresOptions(1e-8, 300, 7))
    xg = gather(xs)
    if rank == 0:
        P1g = stiga.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 0.4, 1.0, scaling=D, device=0)
        x1, rep1 = stiga.gmres(A1, P1g, torch.from_numpy(b).cuda(), stiga.GmresOptions(1e-8, 300, 7))
        out["gmres_its"] = rep.iterations
        out["gmres_its_single"] = rep1.iterations
        out["gmres_converged"] = rep.converged
        out["gmres_x_vs_single"] = rel(xg, x1.cpu().numpy())
        if case == "spacetime":
            Ao = okr.KronSumOperator(pc.dims, oasm.kron_sum_terms(K, M, Wt, Mt, 1.0, 1.0))
            Pog = ofd.ExtendedFDPreconditioner.setup(K, M, Wt, Mt, 0.4, 1.0, scaling=D)
            xo, repo = ogm.gmres(Ao.apply, Pog.apply, b, 1e-8, 300, 7)
            out["gmres_its_oracle"] = repo.iterations
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
