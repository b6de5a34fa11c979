"""Benchmark of the extended-FD preconditioner apply (+ GMRES time-to-1e-8) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5p5] [--impl ours|reference]

One step = one ExtendedFDPreconditioner::apply (fdsolve.cpp:155-164) of the A^G preconditioner
over one seeded uniform[-1,1] vector of the configuration.  Default: the largest single-GPU BASELINE
configuration, c5p5 (configs[4]: d = 3, p = 5, n_el = 160, 710,242,508 DoF, 5.7 GB per vector).
Inputs are resident in HBM and larger than L2 (126 MB), so no L2 flush is needed between steps.
Prints ONE JSON line (rank 0).  --gpus N > 1 without a launcher starts N ranks itself
(torch.distributed.run, 127.0.0.1) and runs the time-sharded apply (strong scaling, same config).

--impl reference times the reference's CPU path for the same workload: the Eigen-free restatement
in oracle/ (the reference itself needs Eigen and cannot be compiled here), each
step a bounded sample of the full apply (oracle/sampled.py).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FD preconditioner applies/s & DoF/s (frac. FP64/HBM roofline); GMRES time-to-1e-8"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5p5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--cpu-frac", type=float, default=None,
                    help="fraction of every pass's units in one sampled CPU apply (default: sized to ~2 s)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 time-sharded apply: p2p = all-to-all fused into the kernels' scatter epilogues "
                         "over NVLink peer memory (CUDA IPC); nccl = pack + NCCL all_to_all_single + unpack")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the time-sharded apply")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------
# clocks sampler (NVML, during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# CPU path (oracle restatement of the reference) -- baseline and --impl reference
# ------------------------------------------------------------------------------------------
def cpu_sampler(cfg, frac=None, target_s=2.0):
    """oracle.sampled.SampledFD for cfg (host pieces of the same workload; c4's geometry pieces come
    from the product's host setup, the timed apply is the oracle's).  frac=None sizes the sample so
    one sampled apply takes ~target_s on all host cores."""
    from oracle.sampled import SampledFD

    pieces = None
    if cfg.problem != "identity":
        pc, _ = problem_pieces(cfg)
        pieces = (pc.K, pc.M, pc.Wt, pc.Mt)
    f = frac if frac is not None else min(1.0, 0.05 * 17.0e6 / cfg.n_dof)
    S = SampledFD(cfg, f, pieces)
    if frac is None:  # rescale from one timed sample
        est, wall, _ = S.run()
        f2 = min(1.0, max(1e-4, f * target_s / max(wall, 1e-3)))
        if abs(f2 - f) / f > 0.3:
            S = SampledFD(cfg, f2, pieces)
    return S


def cpu_baseline(cfg, frac=None):
    """cpu_baseline of the JSON line: the oracle port on a bounded sample, all host cores (OpenBLAS
    threads) and 1 core, plus the CPU GMRES estimate (n_P P + n_A A applies of the identity-geometry
    solve, one iteration: gmres.cpp:42, 76)."""
    from oracle.sampled import SampledMatvec, blas_threads, threads_limit

    S = cpu_sampler(cfg, frac)
    S.run()  # warm-up (study.cpp:210-213 excludes one warm-up apply)
    ests = [S.run()[0] for _ in range(3)]
    t_all = statistics.median(ests)
    cores = blas_threads()
    with threads_limit(1):
        S1 = S if S.frac <= 0.02 else type(S)(cfg, max(1e-4, S.frac / 4), (S.K, S.M, S.Wt, S.Mt))
        S1.run()
        t_one = statistics.median([S1.run()[0] for _ in range(2)])
    out = {"value": 1.0 / t_all, "unit": "applies/s", "cores": cores, "kind": "port",
           "sample": f"oracle/fdsolve.py apply of {cfg.name} (fdsolve.cpp:155-164), every pass on "
                     f"{100 * S.frac:.2f}% of its independent units (slabs / columns / spatial indices) and "
                     f"extrapolated; median of 3 after 1 warm-up; numpy/OpenBLAS on {cores} threads",
           "single_core": {"value": 1.0 / t_one, "unit": "applies/s", "cores": 1,
                           "sample": f"same, {100 * S1.frac:.2f}% of the units, BLAS limited to 1 thread "
                                     f"(the reference is single-threaded, PAPER.md:1120)"},
           "apply_s_all_cores": t_all, "apply_s_single_core": t_one}
    if cfg.problem == "identity":
        A = SampledMatvec(S, S.frac)
        t_a = statistics.median([A.run() for _ in range(2)])
        out["gmres_cpu_est"] = {"time_s": 2 * t_all + t_a, "n_P": 2, "n_A": 1, "matvec_s": t_a,
                                "note": "one-iteration solve (identity geometry): P b, A v_0, P(A v_0); "
                                        "mat-vec = sparse banded Kronecker factors (kronop.cpp:7-41) on the "
                                        "same sampling; Krylov vector updates excluded"}
    return out


def problem_pieces(cfg, device=None):
    """1D factors + D of the A^G preconditioner: identity geometry for c1/c2/c3/c5 (D = 1), the
    fitted deformed cube with kappa(x), c(x) for c4 (BASELINE configs[3]).  With a device, D =
    diag(A)/diag(A~) is formed on the device (stiga_geometry_scaling_device; diag(A) of the
    device-assembled physical operator for c4) and stays there as a CUDA tensor."""
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.problems import Problem, geometry_scaling, identity_pieces

    if cfg.problem == "identity":
        pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
        if device is None:
            return pc, geometry_scaling(pc)
        A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, pc.gamma, pc.nu, device=device)
        At = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=device)
        return pc, stiga.geometry_scaling_device(A, At)
    pc = Problem(cfg.problem).geometry_pieces(cfg.p, cfg.n_el, want_D=True, device=device,
                                              D_on_device=device is not None)
    if hasattr(pc, "A"):
        del pc.A  # the GMRES section builds (and times) its own operator
    return pc, pc.D


def problem_pieces_slab(cfg, world, rank, device=None):
    """problem_pieces for one rank of the time-sharded run: the 1D factors and D on the rank's time slab
    only (per-rank host and device memory ~ N_dof / world)."""
    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.problems import Problem, geometry_scaling, identity_pieces

    n_t = cfg.n_t
    t0, ntl = stiga.shard_partition(n_t, world, rank)
    if cfg.problem == "identity":
        pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
        return pc, geometry_scaling(pc, t_range=(t0, t0 + ntl)), (t0, ntl)
    pc = Problem(cfg.problem).geometry_pieces(cfg.p, cfg.n_el, want_D=True, device=device)
    if hasattr(pc, "A"):
        del pc.A
    n_s = pc.n_dof // n_t
    return pc, pc.D[n_s * t0:n_s * (t0 + ntl)].copy(), (t0, ntl)


def run_reference(args):
    """The reference arm: the oracle port of the reference's CPU path on the box's host cores (all
    BLAS threads), on our arm's config / metric / unit; each step one bounded sample of the full apply
    (oracle/sampled.py), extrapolated to applies/s.  Rank 0 only under a launcher."""
    from oracle.sampled import blas_threads
    from paper_1909_07309_b200.configs import CONFIGS

    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    warm, steps = max(args.warmup, 3), max(1, args.steps)
    t0 = time.perf_counter()
    S = cpu_sampler(cfg, args.cpu_frac, target_s=min(2.0, 150.0 / (warm + steps)))
    setup_s = time.perf_counter() - t0
    for _ in range(warm):
        S.run()
    ests, walls = [], []
    for _ in range(steps):
        e, w, _ = S.run()
        ests.append(e)
        walls.append(w)
    t = sum(ests) / len(ests)
    v = 1.0 / t
    cores = blas_threads()
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "applies/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * t, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1])",
        "dof_per_s": v * cfg.n_dof, "setup_s": setup_s,
        "config": {"workload": f"{cfg.name}: {cfg.note}; A^G FD apply (D^-1/2 scaled), {cfg.problem} geometry",
                   "d": cfg.d, "p": cfg.p, "n_el": cfg.n_el, "n_dof": cfg.n_dof, "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "applies/s", "cores": cores, "kind": "port",
                         "sample": f"each step: every pass of the oracle apply (oracle/fdsolve.py = fdsolve.cpp:155-164) "
                                   f"on {100 * S.frac:.2f}% of its independent units, extrapolated "
                                   f"(sample wall {1e3 * sum(walls) / len(walls):.0f} ms per step; ms_per_step is "
                                   f"the extrapolated full apply)"},
        "e2e": {"value": v, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# GPU path
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1909_07309_b200 import stiga
    from paper_1909_07309_b200.configs import CONFIGS
    from paper_1909_07309_b200.inputs import uniform_pm1
    ws, rank, local = dist_env()
    if os.environ.get("STIGA_BENCH_BACKEND") == "gloo":
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        # STIGA_BENCH_BACKEND=gloo: plumbing check of the N > 1 path with several ranks on one GPU
        # (no NCCL); the fused exchange then uses host barriers
        if os.environ.get("STIGA_BENCH_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    cfg = CONFIGS[args.config]
    K_steps, W_steps = args.steps, max(args.warmup, 3)
    sharded = ws > 1 and not args.replicas
    exchange = None

    t0 = time.perf_counter()
    if sharded:  # this rank's time slab only: the pieces are 1D factors, D is built for the slab
        comm = stiga.Comm.from_process_group(device=dev)
        pc, D, (t_lo, t_len) = problem_pieces_slab(cfg, ws, rank, device=local)
    else:
        pc, D = problem_pieces(cfg, device=local)
    pieces_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    if sharded and args.exchange == "p2p":
        # native time-sharded handle (C ABI): all-to-all fused into the scatter epilogues over CUDA-IPC
        # peer buffers, stream-ordered NCCL barriers between the stages
        P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, comm=comm)
        exchange = "native C ABI: scatter epilogues into peer buffers (CUDA IPC / NVLink), " + \
                   ("NCCL stream-ordered barriers" if dist.get_backend() == "nccl" else "host barriers (gloo)")
    else:
        P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0,
                                                 scaling=D if not sharded else None, device=dev,
                                                 device_schur=True)
    setup_s = time.perf_counter() - t0
    n = P.n_dof
    launches = P.launches()

    if sharded and args.exchange == "p2p":
        a0, a1 = P.local_slice()
        r_host = torch.from_numpy(uniform_pm1(a1 - a0, cfg.seed, start=a0)).pin_memory()
        apply_fn = lambda x, y: P.apply(x, out=y)  # noqa: E731
    elif sharded:  # --exchange nccl: pack + NCCL all_to_all_single + unpack (the Python baseline path)
        from paper_1909_07309_b200.distributed import DeviceBackend, ShardedExtendedFD

        sh = ShardedExtendedFD(DeviceBackend(P), P.dims)
        exchange = "nccl all_to_all_single (pack / unpack), unscaled"
        a0, a1 = sh.plan.local_slice()
        r_host = torch.from_numpy(uniform_pm1(a1 - a0, cfg.seed, start=a0)).pin_memory()
        apply_fn = lambda x, y: sh.apply(x, out=y)  # noqa: E731
    else:
        r_host = torch.from_numpy(uniform_pm1(n, cfg.seed + rank)).pin_memory()
        apply_fn = lambda x, y: P.apply(x, out=y)  # noqa: E731
    s_host = torch.empty_like(r_host).pin_memory()
    r = r_host.cuda(dev)
    s = torch.empty_like(r)
    stream = torch.cuda.current_stream(dev)

    peak_dmma, peak_dfma = stiga.fp64_peak(dev, 300.0)

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        on_cpu = os.environ.get("STIGA_BENCH_BACKEND") == "gloo"
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if on_cpu else f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(W_steps):
        apply_fn(r, s)
    torch.cuda.synchronize()

    # ---- timed region: K device-resident applies --------------------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(dev)
    barrier()
    torch.cuda.synchronize()
    prof_range = os.environ.get("STIGA_PROFILE_RANGE") == "1"  # ncu --profile-from-start off: timed steps only
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    with sampler:
        ev0.record(stream)
        for _ in range(K_steps):
            apply_fn(r, s)
        ev1.record(stream)
        torch.cuda.synchronize()
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / K_steps)
    value = (1 if sharded else ws) / (ms * 1e-3)

    # ---- per-launch durations (separate profiled pass over K steps, events on the same stream) --
    pass_ms = np.zeros(launches)
    kp = min(K_steps, 50)
    rp, sp = (r, s) if (not sharded or args.exchange == "p2p") else (
        torch.zeros(n, dtype=torch.float64, device=f"cuda:{dev}"), torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}"))
    for _ in range(kp):
        pass_ms += np.array(P.apply_profiled(rp, sp))
    pass_ms /= kp
    info = P.launch_info()
    names = [nm for nm, _ in info]
    flops = [fl for _, fl in info]
    dom = int(np.argmax(pass_ms))
    achieved = flops[dom] / (pass_ms[dom] * 1e-3) / 1e12
    traffic = None
    tf_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf_path):
        try:
            traffic = json.load(open(tf_path)).get(cfg.name, {}).get(names[dom])
        except Exception:
            traffic = None

    # ---- e2e: host buffers through the public API, copies inside the timed region -----------------
    # Every step copies its input from pinned host memory (H2D), applies, and reads the result back
    # (D2H).  Steps are software-pipelined over three streams with two device buffer pairs: the copy
    # engines move step k+1's input and step k-1's result while step k computes (the apply itself
    # stays on one stream, so the handle's scratch is never shared).  The serial variant (copy,
    # apply, copy on one stream) is reported alongside.
    ke = max(3, min(K_steps, 50))

    def e2e_serial():
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(ke):
            r.copy_(r_host, non_blocking=True)
            apply_fn(r, s)
            s_host.copy_(s, non_blocking=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / ke)

    r_dev = [r, torch.empty_like(r)]
    s_dev = [s, torch.empty_like(s)]
    s_hosts = [s_host, torch.empty_like(s_host).pin_memory()]
    st_h2d, st_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    mk = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
    ev_h, ev_c, ev_d = mk(), mk(), mk()

    def e2e_pipelined(steps):
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        st_h2d.wait_event(ev0)
        st_d2h.wait_event(ev0)
        for k in range(steps):
            b = k % 2
            with torch.cuda.stream(st_h2d):
                if k >= 2:
                    st_h2d.wait_event(ev_c[b])  # step k-2 is done reading r_dev[b]
                r_dev[b].copy_(r_host, non_blocking=True)
                ev_h[b].record(st_h2d)
            stream.wait_event(ev_h[b])
            if k >= 2:
                stream.wait_event(ev_d[b])  # step k-2's result left s_dev[b]
            apply_fn(r_dev[b], s_dev[b])
            ev_c[b].record(stream)
            with torch.cuda.stream(st_d2h):
                st_d2h.wait_event(ev_c[b])
                s_hosts[b].copy_(s_dev[b], non_blocking=True)
                ev_d[b].record(st_d2h)
        stream.wait_stream(st_d2h)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / steps)

    e2e_pipelined(2)
    e2e_serial_ms = e2e_serial()
    e2e_ms = e2e_pipelined(ke)

    # ---- GMRES time-to-1e-8 (device resident, restart 50, x0 = 0) -----------------------------
    gm = None
    if not args.no_gmres and not sharded:
        t_a = time.perf_counter()
        if cfg.problem == "identity":  # A = kron_sum_terms form, equal to the physical A on F = id
            A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=dev)
        else:  # physical K_s, M_s of the curved geometry assembled on the device
            from paper_1909_07309_b200.problems import Problem

            A = stiga.KronSumOperator.physical(Problem(cfg.problem), cfg.p, cfg.n_el, device=dev)
        torch.cuda.synchronize()
        a_setup_s = time.perf_counter() - t_a
        torch.cuda.synchronize()
        x, rep = stiga.gmres(A, P, r, stiga.GmresOptions(tol=1e-8, max_krylov=500, restart=50))
        torch.cuda.synchronize()
        x, rep = stiga.gmres(A, P, r, stiga.GmresOptions(tol=1e-8, max_krylov=500, restart=50))
        res = (torch.linalg.norm(A.apply(x) - r) / torch.linalg.norm(r)).item()
        ev0.record(stream)
        for _ in range(5):
            A.apply(r, out=s)
        ev1.record(stream)
        torch.cuda.synchronize()
        gm = {"time_s": rep.wall_time_s, "iterations": rep.iterations, "converged": rep.converged,
              "operator_setup_s": a_setup_s, "matvec_ms": ev0.elapsed_time(ev1) / 5,
              "final_rel_precond_residual": rep.residual_history[-1], "true_rel_residual": res,
              "precond_time_fraction": rep.precond_time_fraction, "restart": 50, "tol": 1e-8}
        del A
    elif not args.no_gmres and sharded:  # collective GMRES on the native time-sharded handles (CGS2)
        try:
            t_a = time.perf_counter()
            if args.exchange != "p2p":
                raise RuntimeError("the GMRES section needs the native sharded handles (--exchange p2p)")
            if cfg.problem == "identity":
                A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, comm=comm)
            else:
                from paper_1909_07309_b200.problems import Problem

                A = stiga.KronSumOperator.physical(Problem(cfg.problem), cfg.p, cfg.n_el, comm=comm)
            torch.cuda.synchronize()
            a_setup_s = time.perf_counter() - t_a
            opts = stiga.GmresOptions(tol=1e-8, max_krylov=500, restart=50)
            x, rep = stiga.gmres(A, P, r, opts)
            barrier()
            x, rep = stiga.gmres(A, P, r, opts)
            res_v = A.apply(x) - r
            nums = torch.stack([torch.dot(res_v, res_v), torch.dot(r, r)])
            comm.allreduce(nums)
            res = (nums[0] / nums[1]).sqrt().item()
            ev0.record(stream)
            for _ in range(5):
                A.apply(r, out=s)
            ev1.record(stream)
            torch.cuda.synchronize()
            gm = {"time_s": max_over_ranks(rep.wall_time_s), "iterations": rep.iterations,
                  "converged": rep.converged, "operator_setup_s": a_setup_s,
                  "matvec_ms": max_over_ranks(ev0.elapsed_time(ev1) / 5),
                  "final_rel_precond_residual": rep.residual_history[-1], "true_rel_residual": res,
                  "restart": 50, "tol": 1e-8, "sharded": f"time x{ws} (native C ABI, halo push over CUDA IPC)",
                  "ortho": "CGS2, batched dots (two all-reduces per Arnoldi column)"}
            del A
        except Exception as e:  # report, do not lose the apply numbers
            gm = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_frac)

    f_alg = cfg.flops_fd()
    g_eff = ws if sharded else 1  # the sharded job's roofline is the N-GPU one
    t_roof_flop = f_alg / (g_eff * peak_dmma * 1e12)
    t_roof_hbm = 32.0 * n / (g_eff * 6538.9e9)
    out = {
        "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": ws, "steps": K_steps, "warmup": W_steps,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1], splitmix64)",
        "config": {"workload": f"{cfg.name}: {cfg.note}; A^G FD apply (D^-1/2 scaled), {cfg.problem} geometry",
                   "d": cfg.d, "p": cfg.p, "n_el": cfg.n_el, "n_dof": n, "dims": P.dims,
                   "parallelism": (f"time-sharded x{ws} ({exchange})" if sharded else
                                   ("replicas" if ws > 1 else "single")),
                   "l2": "inputs (136 MB+) larger than L2 (126 MB); no flush"},
        "dof_per_s": value * n,
        "apply_roofline": {"F_alg_flop": f_alg, "t_roof_ms": 1e3 * max(t_roof_flop, t_roof_hbm),
                           "frac": max(t_roof_flop, t_roof_hbm) / (ms * 1e-3), "peak_tflops": peak_dmma,
                           "bound": "fp64 (DMMA)",
                           "F_exec_flop": float(sum(flops)),
                           "frac_exec": float(sum(flops)) / (peak_dmma * 1e12) / (ms * 1e-3),  # per rank
                           "note": "F_alg = 4 N (sum n_l + n_t) (PAPER.md:1061-1064, dense mode products); "
                                   "F_exec = FP64 work the launches execute (a folded centrosymmetric product "
                                   "does ~half of a dense one, DESIGN.md §5)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_dmma, "unit": "TFLOP/s",
                     "frac": achieved / peak_dmma, "traffic": traffic, "kernel": names[dom],
                     "flop_per_launch": flops[dom],
                     "peak_source": "FP64 DMMA m8n8k4 probe measured live in this run (MEASURED_PEAKS.json has no FP64)",
                     "peak_dfma_tflops": peak_dfma},
        "pass_ms": {names[i]: float(pass_ms[i]) for i in range(launches)},
        "e2e": {"value": (1 if sharded else ws) / (e2e_ms * 1e-3), "unit": "applies/s",
                "h2d_bytes_per_step": 8 * r.numel(), "d2h_bytes_per_step": 8 * r.numel(), "ms_per_step": e2e_ms,
                "pipelining": "H2D / apply / D2H on three streams, two buffer pairs",
                "serial_value": (1 if sharded else ws) / (e2e_serial_ms * 1e-3)},
        "gpu_launches": K_steps * (len([nm for nm in names if not nm.startswith("exchange_barrier")]) +
                                   (2 * ws if sharded and exchange.startswith("nccl") else 0)),
        "setup_s": setup_s, "pieces_s": pieces_s,
        "gmres": gm,
        "cpu_baseline": cpu,
        "clocks": sampler.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n):
    """--gpus N > 1 without a launcher: start N ranks (one process per GPU) with torch.distributed.run on
    127.0.0.1 and relay rank 0's line; the exit code is the launcher's."""
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
