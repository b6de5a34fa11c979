"""Committed golden vectors (tests/golden/*.npz, made by tests/golden/make_golden.py from the pinned
oracle): CPU check that the oracle still reproduces them, GPU check of the product against them."""
import glob
import os

import numpy as np
import pytest

from oracle.assembly import assemble_spatial_parametric, assemble_time_matrices
from oracle.fdsolve import ExtendedFDPreconditioner as OracleFD
from paper_1909_07309_b200.inputs import uniform_pm1

FILES = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "*.npz")))


def load(f):
    z = np.load(f)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("f", FILES, ids=[os.path.basename(f) for f in FILES])
def test_oracle_reproduces_golden(f):
    g = load(f)
    d, p, nel = int(g["d"]), int(g["p"]), int(g["n_el"])
    assert np.array_equal(uniform_pm1(len(g["r"]), int(g["seed"])), g["r"])
    W, Mt = assemble_time_matrices(p, nel, 1.0)
    K, M = assemble_spatial_parametric(p, nel, d)
    D = g["scaling"] if g["scaling"].size else None
    s = OracleFD.setup(K, M, W, Mt, 1.0, 1.0, scaling=D).apply(g["r"])
    assert np.linalg.norm(s - g["s"]) <= 1e-12 * np.linalg.norm(g["s"])


@pytest.mark.gpu
@pytest.mark.parametrize("f", FILES, ids=[os.path.basename(f) for f in FILES])
def test_gpu_matches_golden(f):
    torch = pytest.importorskip("torch")
    from paper_1909_07309_b200 import stiga

    g = load(f)
    d, p, nel = int(g["d"]), int(g["p"]), int(g["n_el"])
    W, Mt = stiga.assemble_time_matrices(p, nel, 1.0)
    K, M = stiga.assemble_spatial_parametric(p, nel, d)
    D = g["scaling"] if g["scaling"].size else None
    P = stiga.ExtendedFDPreconditioner.setup(K, M, W, Mt, 1.0, 1.0, scaling=D, device=0)
    s = P.apply(torch.from_numpy(g["r"]).cuda()).cpu().numpy()
    assert np.linalg.norm(s - g["s"]) <= 1e-11 * np.linalg.norm(g["s"])
    A = stiga.KronSumOperator.spacetime(K, M, W, Mt, 1.0, 1.0)
    x, rep = stiga.gmres(A, P, torch.from_numpy(g["r"]).cuda(), stiga.GmresOptions(1e-8, 100, 50))
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert np.linalg.norm(x.cpu().numpy() - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
