"""Small host-stepped runs of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): Burgers 1D (collocated + over-integrated),
2D Burgers, 2D Euler (strip JVP, LF + Roe, CGS2 + DCGS2), 3D Euler, EXPRB42."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import to_dev

kw = dict(use_graph=False)
for orth in ("cgs2", "dcgs2"):
    ctx = pkg.Context(0, orth=orth)
    for w, integ in ((configs.scaled(configs.C1_S3E4, 16, steps=2), "epi2"),
                     (configs.scaled(configs.C3, 6, steps=1), "epi2"),
                     (configs.scaled(configs.C4, 12, steps=1), "epi2"),
                     (configs.scaled(configs.C4, 12, steps=1), "exprb42"),
                     (configs.scaled(configs.C5, 4, steps=1), "epi2")):
        u0 = w.initial_condition()
        dt = w.time_step(u0) if w.dt is None else w.dt
        for flux in (("lf", "roe") if w.spec().kind == "euler2d" else (None,)):
            spec = w.spec()
            if flux:
                spec.euler_flux = flux
            op = pkg.Operator(ctx, spec)
            r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, w.steps * dt, tol=w.tol, max_basis=w.max_basis,
                              orth_length=w.max_basis, **kw)
            print(orth, w.name, integ, flux, r.status, r.steps, r.krylov_iterations, flush=True)
    spec = pkg.OperatorSpec("burgers1d", 3, 12, box=(0, 1, 0, 1, 0, 1), periodic=False, kappa=0.03, flux="ef",
                            sigma=1e-3, over_integrate=True)
    op = pkg.Operator(ctx, spec)
    op.set_source_function(lambda x: 0.1 * x)
    import numpy as np
    u0 = np.sin(np.linspace(0, 3, op.dim))
    r = pkg.integrate(ctx, op, to_dev(u0), "exprb32", 1e-3, 3e-3, tol=1e-10, max_basis=30, orth_length=30, **kw)
    print(orth, "burgers-oi", r.status, r.steps, flush=True)
print("sanitize run done")
