"""The NATIVE multi-GPU path through the C ABI (include/stiga_gpu.h "multi-GPU"): communicator,
time-sharded FD apply with the all-to-all fused into the scatter epilogues (CUDA IPC peer buffers),
time-sharded system mat-vec with the halo push, collective GMRES (CGS2) -- run with 2 and 3 ranks
sharing this one GPU over a gloo-backed host-callback communicator (tests/_native_sharded_worker.py).
Parity against the single-device product and the oracle; per-rank device memory ~ N_dof / world."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_ranks(world, case):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "_native_sharded_worker.py"), case]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    errs = [ln for ln in out.stderr.splitlines() if "Error" in ln or "error" in ln][:20]
    assert out.returncode == 0, ("\n".join(errs), out.stdout[-2000:], out.stderr[-3000:])
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("world", [2, 3])
def test_native_sharded_spacetime(world):
    d = run_ranks(world, "spacetime")
    assert d["apply_vs_oracle"] <= 1e-11 and d["apply_vs_single"] <= 1e-13
    assert "exchange_barrier_1" in d["launches"] and d["profiled_ok"]
    assert d["matvec_vs_oracle"] <= 1e-12 and d["matvec_vs_single"] <= 1e-14 and d["matvec_repeat_equal"]
    assert d["gmres_converged"] and d["gmres_its"] > 3
    assert abs(d["gmres_its"] - d["gmres_its_oracle"]) <= 1 and abs(d["gmres_its"] - d["gmres_its_single"]) <= 1
    assert d["gmres_x_vs_single"] <= 1e-6


def test_native_sharded_physical():
    d = run_ranks(2, "physical")
    assert d["apply_vs_oracle"] <= 1e-11 and d["apply_vs_single"] <= 1e-13
    assert d["matvec_vs_single"] <= 1e-13 and d["matvec_repeat_equal"]
    assert d["gmres_converged"] and abs(d["gmres_its"] - d["gmres_its_single"]) <= 1


def test_native_sharded_memory_per_rank():
    """Per-rank device memory of a sharded FD handle ~ N_dof / world: two scratch slabs, two receive
    buffers and the D^-1/2 slab (5 N_dof / world doubles) plus the factors -- not the full-size
    scratch and D of a single-device handle (c2 size, 17M DoF)."""
    d = run_ranks(2, "memory")
    n = d["n_dof"]
    per_rank = d["fd_bytes_all_ranks"] / 2
    assert per_rank <= 8 * 5.5 * n / 2 + 64e6, (per_rank, n)
    assert d["fd_bytes_single"] >= 8 * 3 * n  # in/out scratch + D^-1/2, full size
    assert d["apply_vs_single"] <= 1e-13
