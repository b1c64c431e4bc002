"""Small host-stepped runs of the role-split (face-warp) JVP kernels and the cluster engine for
compute-sanitizer (racecheck / memcheck / synccheck): pipelined DCGS2 on C4 (partial strips, Roe),
C5 (partial tiles, order 1 and 3) and the C1 cluster engine."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402
from tests.gpu_util import to_dev  # noqa: E402
from tests.test_gpu_euler2d import random_state  # noqa: E402
from tests.test_gpu_extensions import random_state5  # noqa: E402

rng = np.random.default_rng(3)
ctx = pkg.Context(0, orth="dcgs2", fused=False)
kw = dict(tol=1e-10, max_basis=8, orth_length=8, use_graph=False)
for order, nx, ny, flux in ((4, 7, 3, "lf"), (4, 6, 2, "roe"), (2, 9, 2, "lf")):
    spec = pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), euler_flux=flux)
    r = pkg.integrate(ctx, pkg.Operator(ctx, spec), to_dev(random_state(rng, nx * ny, (order + 1) ** 2)), "epi2",
                      2e-4, 2e-4, **kw)
    print("euler2d", order, nx, ny, flux, r.status, r.krylov_iterations, ctx.last_path(), flush=True)
for order, dims in ((3, (3, 2, 3)), (1, (5, 9, 2))):
    nx, ny, nz = dims
    spec = pkg.OperatorSpec("euler3d", order, nx, ny, nz, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    r = pkg.integrate(ctx, pkg.Operator(ctx, spec), to_dev(random_state5(rng, nx * ny * nz, (order + 1) ** 3)),
                      "epi2", 2e-4, 2e-4, **kw)
    print("euler3d", order, dims, r.status, r.krylov_iterations, ctx.last_path(), flush=True)
c1 = pkg.Context(0)
w = configs.scaled(configs.C1_S3E4, 32, steps=2)
r = pkg.integrate(c1, pkg.Operator(c1, w.spec()), to_dev(w.initial_condition()), "epi2", w.dt, 2 * w.dt, tol=w.tol,
                  max_basis=w.max_basis, orth_length=w.max_basis)
print("C1 cluster", r.status, r.krylov_iterations, c1.last_path(), flush=True)
print("sanitize run done")
