"""Benchmark of the extended-FD preconditioner apply (+ GMRES time-to-1e-8) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one ExtendedFDPreconditioner::apply (fdsolve.cpp:155-164) of the A^G preconditioner
over one seeded uniform[-1,1] vector of the configuration (BASELINE.json configs[1] = c2 by
default: d=2, p=3, n_el=256, 17,040,642 DoF).  Inputs are resident in HBM and larger than L2
(136 MB > 126 MB), so no L2 flush is needed between steps.  Prints ONE JSON line (rank 0).

--impl reference times the reference's CPU path for the same workload: the Eigen-free restatement
in oracle/ (the reference itself needs Eigen and cannot be compiled here).
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
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
def cpu_fd_timing(cfg, steps, warmup, budget_s=None):
    import numpy as np

    from oracle.assembly import assemble_spatial_parametric, assemble_time_matrices
    from oracle.fdsolve import ExtendedFDPreconditioner as OracleFD
    from paper_1909_07309_b200.inputs import uniform_pm1

    if cfg.problem == "identity":
        W, Mt = assemble_time_matrices(cfg.p, cfg.n_el, 1.0)
        K, M = assemble_spatial_parametric(cfg.p, cfg.n_el, cfg.d)
        D = np.ones(cfg.n_dof)  # diag(A)/diag(A~) on the identity map (see problems.geometry_scaling)
    else:  # host pieces (geometry fit, separation, D) from the product's setup code; the apply is timed
        pc, D = problem_pieces(cfg)
        K, M, W, Mt = pc.K, pc.M, pc.Wt, pc.Mt
    t0 = time.perf_counter()
    P = OracleFD.setup(K, M, W, Mt, 1.0, 1.0, scaling=D)
    setup_s = time.perf_counter() - t0
    r = uniform_pm1(cfg.n_dof, cfg.seed)
    for _ in range(warmup):
        P.apply(r)
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        P.apply(r)
        times.append(time.perf_counter() - t0)
        if budget_s is not None and time.perf_counter() - t_start > budget_s:
            break
    return times, setup_s


def problem_pieces(cfg, device=None):
    """1D factors + D of the A^G preconditioner: identity geometry for c1/c2/c3/c5 (D = 1), the
    fitted deformed cube with kappa(x), c(x) for c4 (BASELINE configs[3]).  With a device, diag(A)
    of D comes from the device-assembled physical operator instead of the host quadrature."""
    from paper_1909_07309_b200.problems import Problem, geometry_scaling, identity_pieces

    if cfg.problem == "identity":
        pc = identity_pieces(cfg.d, cfg.p, cfg.n_el)
        return pc, geometry_scaling(pc)
    pc = Problem(cfg.problem).geometry_pieces(cfg.p, cfg.n_el, want_D=True, device=device)
    if hasattr(pc, "A"):
        del pc.A  # the GMRES section builds (and times) its own operator
    return pc, pc.D


def cores_used():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        n = max((i.get("num_threads", 1) for i in info if i.get("user_api") == "blas"), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    from paper_1909_07309_b200.configs import CONFIGS

    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    warm = max(1, min(args.warmup, 3))
    steps = max(1, min(args.steps, 20))
    times, setup_s = cpu_fd_timing(cfg, steps, warm, budget_s=150.0)
    total = sum(times)
    v = len(times) / total
    cores = cores_used()
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "applies/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1])",
        "dof_per_s": v * cfg.n_dof, "setup_s": setup_s,
        "config": {"workload": f"{cfg.name}: {cfg.note}; A^G FD apply", "d": cfg.d, "p": cfg.p, "n_el": cfg.n_el,
                   "n_dof": cfg.n_dof, "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "applies/s", "cores": cores, "kind": "port",
                         "sample": f"{len(times)} full {cfg.name} applies of the numpy/OpenBLAS restatement "
                                   f"(oracle/fdsolve.py, reference fdsolve.cpp:155-164)"},
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

    t0 = time.perf_counter()
    pc, D = problem_pieces(cfg, device=local)
    pieces_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    P = stiga.ExtendedFDPreconditioner.setup(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, scaling=D, device=dev)
    setup_s = time.perf_counter() - t0
    n = P.n_dof
    launches = P.launches()

    sharded = ws > 1 and not args.replicas
    exchange = None
    if sharded:  # time-sharded apply: rank owns a time slab, two all-to-all transposes per apply
        from paper_1909_07309_b200.distributed import DeviceBackend, FusedShardedExtendedFD, ShardedExtendedFD

        sh = None
        if args.exchange == "p2p":
            try:
                sh = FusedShardedExtendedFD.create(P, P.dims, device=dev)
                exchange = "p2p scatter epilogues (CUDA IPC peer memory)"
            except Exception as e:  # e.g. no peer access between these GPUs: keep the NCCL exchange
                exchange = f"nccl (p2p unavailable: {type(e).__name__}: {str(e)[:120]})"
        if sh is None:
            sh = ShardedExtendedFD(DeviceBackend(P), P.dims)
            exchange = exchange or "nccl all_to_all_single (pack / unpack)"
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
    rp, sp = (r, s) if not sharded else (torch.zeros(n, dtype=torch.float64, device=f"cuda:{dev}"),
                                         torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}"))
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
    elif not args.no_gmres and sharded:  # time-sharded GMRES: halo-exchanged A, all-reduced dots
        try:
            from paper_1909_07309_b200.distributed import (DeviceSystemBackend, DeviceVec, ShardedSystem,
                                                           sharded_gmres)

            t_a = time.perf_counter()
            if cfg.problem == "identity":
                A = stiga.KronSumOperator.spacetime(pc.K, pc.M, pc.Wt, pc.Mt, 1.0, 1.0, device=dev)
            else:
                from paper_1909_07309_b200.problems import Problem

                A = stiga.KronSumOperator.physical(Problem(cfg.problem), cfg.p, cfg.n_el, device=dev)
            torch.cuda.synchronize()
            a_setup_s = time.perf_counter() - t_a
            Ash = ShardedSystem(DeviceSystemBackend(A), A.dims)
            vec = DeviceVec()
            x, rep = sharded_gmres(Ash, sh, r, vec, 1e-8, 500, 50, ortho="cgs2")
            barrier()
            x, rep = sharded_gmres(Ash, sh, r, vec, 1e-8, 500, 50, ortho="cgs2")
            res_v = Ash.apply(x)
            vec.axpy(-1.0, r, res_v)
            res = (vec.dot(res_v, res_v) / vec.dot(r, r)) ** 0.5
            gm = {"time_s": max_over_ranks(rep.wall_time_s), "iterations": rep.iterations,
                  "converged": rep.converged, "operator_setup_s": a_setup_s,
                  "final_rel_precond_residual": rep.residual_history[-1], "true_rel_residual": res,
                  "restart": 50, "tol": 1e-8, "sharded": f"time x{ws}",
                  "ortho": "CGS2, batched dots (two all-reduces per Arnoldi column)"}
            del A, Ash
        except Exception as e:  # report, do not lose the apply numbers
            gm = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        times, _ = cpu_fd_timing(cfg, 100, 1, budget_s=args.cpu_budget_s)
        cpu = {"value": len(times) / sum(times), "unit": "applies/s", "cores": cores_used(), "kind": "port",
               "sample": f"{len(times)} full {cfg.name} applies (after 1 warm-up) of the numpy/OpenBLAS restatement "
                         f"oracle/fdsolve.py of fdsolve.cpp:155-164"}

    f_alg = cfg.flops_fd()
    t_roof_flop = f_alg / (peak_dmma * 1e12)
    t_roof_hbm = 32.0 * n / 6538.9e9
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
                           "frac_exec": float(sum(flops)) / (peak_dmma * 1e12) / (ms * 1e-3),
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
        "gpu_launches": K_steps * (launches + (2 * ws if sharded and exchange.startswith("nccl") else 0)),
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


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
