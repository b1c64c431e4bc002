"""Debug: criterion-5 problem (burgers-smooth k=4 ne=40 EF sigma 3e-4, EPI2 dt 0.1) under CGS2 and DCGS2."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle
import paper_2011_01316_b200 as pkg
from tests.gpu_util import to_dev, to_host

u0, src, cfg = oracle.harness_burgers("burgers-smooth", 40, 4, sys.argv[1] if len(sys.argv) > 1 else "ef",
                                      float(sys.argv[2]) if len(sys.argv) > 2 else 3e-4)
ctx = pkg.Context(0)
spec = pkg.OperatorSpec("burgers1d", 4, 40, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                        flux=cfg["flux"], sigma=cfg["sigma"], sigma_adaptive=cfg["sigma_adaptive"],
                        over_integrate=cfg["over_integrate"])
op = pkg.Operator(ctx, spec)
dt = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
u = to_dev(u0)
op.linearize(u)
for step in range(3):
    try:
        u2, st = pkg.step_epi2(ctx, op, u.clone(), dt, tol=1e-12, max_basis=128, orth_length=128)
        print("step", step, "iters", st.iterations, "substeps", st.substeps, "max", float(u2.abs().max()))
        u = u2
        op.linearize(u)
    except Exception as e:
        print("step", step, "error", type(e).__name__, e, ctx.debug_state())
        break
