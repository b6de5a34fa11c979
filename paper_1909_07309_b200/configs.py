"""BASELINE.json configurations (c1..c5) and their derived sizes.

n_s = n_el + p - 2 per spatial direction (both ends dropped), n_t = n_el + p - 1 (t = 0 dropped),
bspline.cpp:139-145.  Config 4 is the fitted deformed cube with variable conductivity / capacity (problems.Problem)."""
from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    d: int
    p: int
    n_el: int
    seed: int
    note: str = ""
    problem: str = "identity"  # "identity" or a Problem id (c4: "deformed-cube-3d")

    @property
    def n_s(self):
        return self.n_el + self.p - 2

    @property
    def n_t(self):
        return self.n_el + self.p - 1

    @property
    def n_dof(self):
        return self.n_s ** self.d * self.n_t

    def flops_fd(self):
        """F_alg = 4 N_dof (d n_s + n_t)."""
        return 4 * self.n_dof * (self.d * self.n_s + self.n_t)


CONFIGS = {
    "c1": Config("c1", 2, 2, 16, 1, "d2 p2 n16 (CPU-runnable reference case)"),
    "c2": Config("c2", 2, 3, 256, 2, "d2 p3 n256 (~17M DoF)"),
    "c3": Config("c3", 3, 3, 96, 3, "d3 p3 n96 (~9e7 DoF)"),
    "c4": Config("c4", 3, 4, 64, 4, "d3 p4 n64 deformed cube, kappa(x), c(x)", "deformed-cube-3d"),
    "c5p2": Config("c5p2", 3, 2, 64, 5, "sweep p2 n64"),
    "c5p3": Config("c5p3", 3, 3, 96, 5, "sweep p3 n96"),
    "c5p4": Config("c5p4", 3, 4, 128, 5, "sweep p4 n128"),
    "c5p5": Config("c5p5", 3, 5, 160, 5, "sweep p5 n160"),
}
