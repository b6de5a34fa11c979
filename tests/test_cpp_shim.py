"""The C++ drop-in binding (include/stiga_b200.hpp, the shim INTEGRATION.md describes) compiled into
a C++ executable linked against libstiga_gpu.so: builds here with g++ (CPU), and on the GPU it runs
the c1 golden parity (apply with and without D) and GMRES through the library handles, through user
callbacks (stiga_gmres_op) and with a user-composed operator A + sigma I."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1909_07309_b200", "lib")
CUDA = "/usr/local/cuda"


def build(out_dir):
    exe = os.path.join(out_dir, "shim_test")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include", "-L", LIBDIR, "-lstiga_gpu",
           f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-3000:]
    return exe


def test_cpp_shim_builds():
    with tempfile.TemporaryDirectory() as td:
        assert os.path.exists(build(td))


@pytest.mark.gpu
def test_cpp_shim_parity_and_gmres():
    from oracle import assembly as oasm
    from oracle import fdsolve as ofd
    from oracle import gmres as ogm
    from oracle import kronop as okr

    g = np.load(os.path.join(ROOT, "tests", "golden", "c1.npz"))
    gs = np.load(os.path.join(ROOT, "tests", "golden", "c1_scaled.npz"))
    with tempfile.TemporaryDirectory() as td:
        exe = build(td)
        g["r"].astype(np.float64).tofile(os.path.join(td, "r.bin"))
        D = gs["scaling"]
        D.astype(np.float64).tofile(os.path.join(td, "D.bin"))
        res = subprocess.run([exe, td], capture_output=True, text=True, timeout=300)
        assert res.returncode == 0, res.stderr[-2000:]
        out = json.loads(res.stdout.strip().splitlines()[-1])
        s = np.fromfile(os.path.join(td, "s.bin"))
        ss = np.fromfile(os.path.join(td, "s_scaled.bin"))
        x_cb = np.fromfile(os.path.join(td, "x_cb.bin"))
        x_shift = np.fromfile(os.path.join(td, "x_shift.bin"))
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(s, g["s"]) <= 1e-11
    W, Mt = oasm.assemble_time_matrices(2, 16, 1.0)
    K, M = oasm.assemble_spatial_parametric(2, 16, 2)
    so = ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=D).apply(g["r"])
    assert rel(ss, so) <= 1e-11
    assert out["invalid_argument"]
    # GMRES: native handles == callback operators; iteration counts vs the oracle's gmres.cpp restatement
    Ao = okr.KronSumOperator([16, 16, 17], oasm.kron_sum_terms(K, M, W, Mt, 1.0, 1.0))
    Pg = ofd.ExtendedFDPreconditioner.setup(K, M, W, Mt, 0.4, 1.0)
    xo, repo = ogm.gmres(Ao.apply, Pg.apply, g["r"], 1e-8, 200, 50)
    assert out["native_converged"] and out["cb_converged"] and out["native_its"] > 3
    assert out["cb_its"] == out["native_its"] and out["cb_vs_native"] <= 1e-14
    assert abs(out["native_its"] - repo.iterations) <= 1
    assert rel(x_cb, xo) <= 1e-6
    sigma = out["sigma"]
    xs, reps = ogm.gmres(lambda v: Ao.apply(v) + sigma * v, Pg.apply, g["r"], 1e-8, 200, 50)
    assert out["shift_converged"] and abs(out["shift_its"] - reps.iterations) <= 1
    assert rel(x_shift, xs) <= 1e-6
    # SpaceTimeSystem through the C++ binding: annulus, A-hat-G with device D, device RHS, errors
    from oracle import problems as opr

    prob = opr.make_full_problem("quarter-annulus-2d")
    sysm = opr.SpaceTimeSystem(prob, 2, 8)
    x, rep = sysm.solve(sysm.make_geometry_preconditioner(), tol=1e-10, max_krylov=300)
    eo = opr.compute_errors(x, sysm.spaces, sysm.tspace, prob, 5)
    assert out["sys_n"] == sysm.n_dof and out["sys_converged"]
    assert abs(out["sys_its"] - rep.iterations) <= 1
    assert abs(out["err_l2l2"] - eo[0]) <= 1e-6 * eo[0] and abs(out["err_x"] - eo[1]) <= 1e-6 * eo[1]
    assert abs(out["gamma_mean"] - sysm.gamma_mean) <= 1e-14 and abs(out["nu_mean"] - sysm.nu_mean) <= 1e-13
