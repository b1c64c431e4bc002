"""BASELINE.json configs C1-C5 as runnable workloads.

All inputs are seeded synthetic data (splitmix64 -> Box-Muller); the seeds are
fixed here so the oracle and the device consume the same bytes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

SEEDS = {1: 20201103, 2: 20201104, 3: 20201105, 4: 20201106, 5: 0}


@dataclass
class Workload:
    name: str
    config: int          # 1..5 (IC generator id)
    kind: str
    order: int
    nx: int
    ny: int = 1
    nz: int = 1
    box: tuple = (0.0, 1.0, 0.0, 1.0, 0.0, 1.0)
    periodic: bool = True
    kappa: float = 0.03
    flux: str = "lf"
    sigma: float = 0.0
    euler_flux: str = "lf"
    dt: Optional[float] = None  # None: Cr_a = cfl from the initial state (C4/C5 rule)
    cfl: float = 5.0
    steps: int = 1
    tol: float = 1e-10
    max_basis: int = 30
    noise: float = 0.0
    gamma: float = 1.4

    def spec(self):
        from . import OperatorSpec
        return OperatorSpec(kind=self.kind, order=self.order, nx=self.nx, ny=self.ny, nz=self.nz, box=self.box,
                            periodic=self.periodic, kappa=self.kappa, flux=self.flux, sigma=self.sigma,
                            euler_flux=self.euler_flux, gamma=self.gamma)

    def initial_condition(self):
        from . import initial_condition
        if self.config == 5 and not (self.nx == self.ny == self.nz):
            return self.initial_condition_slab(0, self.nz)
        return initial_condition(self.config, self.nx, self.order, SEEDS[self.config], self.noise)

    def initial_condition_slab(self, layer_begin: int, layer_end: int):
        """The owned z-slab of a z-partitioned C5 run (no rank builds the global state)."""
        from . import initial_condition_slab
        if self.config != 5:
            raise ValueError("initial_condition_slab: config 5 only (slice the global state otherwise)")
        return initial_condition_slab(5, self.nx, self.ny, self.nz, self.order, layer_begin, layer_end, self.box)

    @property
    def dofs(self) -> int:
        npe = (self.order + 1) ** {"burgers1d": 1, "burgers2d": 2, "euler2d": 2, "euler3d": 3}[self.kind]
        comps = {"burgers1d": 1, "burgers2d": 1, "euler2d": 4, "euler3d": 5}[self.kind]
        return self.nx * self.ny * self.nz * npe * comps

    def time_step(self, u0=None, nodes=None) -> float:
        """dt, or the C4/C5 rule dt = cfl * dx_min / c_max (proj/src/harness.cpp:216-238).
        `nodes`: the LGL nodes of the order (default: the library's host setup; the CPU
        reference arm passes the oracle's, so it never loads the CUDA library)."""
        if self.dt is not None:
            return self.dt
        import numpy as np
        if nodes is None:
            from . import lgl_basis
            nodes = lgl_basis(self.order)[0]
        x = np.asarray(nodes)
        gap = min(2.0, float(np.min(np.diff(x))))
        h = min((self.box[1] - self.box[0]) / self.nx, (self.box[3] - self.box[2]) / self.ny)
        if self.kind == "euler3d":
            h = min(h, (self.box[5] - self.box[4]) / self.nz)
        dx = h * gap / 2.0
        comps = 4 if self.kind == "euler2d" else 5
        npe = (self.order + 1) ** (2 if self.kind == "euler2d" else 3)
        q = u0.reshape(-1, comps, npe)
        rho = q[:, 0]
        vel = [q[:, 1 + d] / rho for d in range(comps - 2)]
        E = q[:, comps - 1]
        p = (self.gamma - 1.0) * (E - 0.5 * rho * sum(v * v for v in vel))
        a = np.sqrt(self.gamma * p / rho)
        c = float(np.max(np.max(np.abs(np.stack(vel)), axis=0) + a))
        return self.cfl * dx / c

    @property
    def t_final(self) -> float:
        return self.steps * self.dt if self.dt is not None else float("nan")


TWO_PI = 2.0 * math.pi

# C1 (configs[0]) — runs on the reference CPU path: entropy flux, sigma = 1.
C1 = Workload("C1-burgers1d-K512-N4", 1, "burgers1d", 4, 512, box=(0.0, TWO_PI, 0, 1, 0, 1), kappa=1e-2,
              flux="ef", sigma=1.0, dt=1e-3, steps=1000, tol=1e-10, max_basis=30)
# C1 with the paper's EF penalty sigma = 3e-4: the labelled
# non-degenerate parity case (C1 itself blows up at step 3 in the reference algorithm).
C1_S3E4 = replace(C1, name="C1s-burgers1d-K512-N4-sigma3e-4", sigma=3e-4)
# C2 (configs[1]) — 1D Burgers at scale (LF, sigma 0: BurgersConfig defaults).
C2 = Workload("C2-burgers1d-K2^20-N7", 2, "burgers1d", 7, 1 << 20, box=(0.0, TWO_PI, 0, 1, 0, 1), kappa=1e-4,
              flux="lf", dt=1e-4, steps=200, tol=1e-10, max_basis=30)
# C3 (configs[2]) — 2D Burgers, not in the reference (tensor-product extension).
C3 = Workload("C3-burgers2d-512^2-N4", 3, "burgers2d", 4, 512, 512, box=(0.0, 1.0, 0.0, 1.0, 0, 1), kappa=1e-3,
              flux="lf", dt=5e-4, steps=100, tol=1e-10, max_basis=30)
# C4 (configs[3]) — 2D Euler strength-5 vortex, LF, Cr_a = 5.
C4 = Workload("C4-euler2d-vortex-1024^2-N4", 4, "euler2d", 4, 1024, 1024, box=(0.0, 10.0, 0.0, 10.0, 0, 1),
              dt=None, cfl=5.0, steps=100, tol=1e-10, max_basis=40, noise=1e-6)
# C5 (configs[4]) — 3D Euler Taylor-Green, 64^3 on one GPU, LF, Cr_a = 5.
C5 = Workload("C5-euler3d-tgv-64^3-N3", 5, "euler3d", 3, 64, 64, 64, box=(0.0, TWO_PI, 0.0, TWO_PI, 0.0, TWO_PI),
              dt=None, cfl=5.0, steps=50, tol=1e-10, max_basis=40)

# C5 at the north star's full size, 128^3 (671,088,640 DOF): z-slab partitioned over 2/4/8 GPUs.
# Memory: ~50 vectors of 5.37 GB (42 Krylov slots at max dim 40, 6 step scratch vectors, the
# frozen primitives, u, the e2e staging copy) = ~270 GB in all, 134 GB per rank at N = 2,
# 67 GB at N = 4, 34 GB at N = 8 -- it does not fit one 180 GB B200.  `bench.py --config C5L
# --nz 32` runs the 128 x 128 x 32 mesh of the same box (one rank's share of the N = 4 job,
# same dt: dx_min is set by the x/y spacing) on one GPU.
C5L = replace(C5, name="C5L-euler3d-tgv-128^3-N3", nx=128, ny=128, nz=128)

ALL = {"C1": C1, "C1s": C1_S3E4, "C2": C2, "C3": C3, "C4": C4, "C5": C5, "C5L": C5L}


def scaled(w: Workload, nx: int, ny: Optional[int] = None, nz: Optional[int] = None, steps: Optional[int] = None):
    """Same physics and Courant rule on a smaller mesh (parity-test sizes)."""
    ny = ny if ny is not None else (nx if w.ny > 1 else 1)
    nz = nz if nz is not None else (nx if w.nz > 1 else 1)
    return replace(w, name=f"{w.name}@{nx}", nx=nx, ny=ny, nz=nz, steps=steps if steps is not None else w.steps)
