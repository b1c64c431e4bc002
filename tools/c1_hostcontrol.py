"""C1 (sigma = 3e-4) a few steps with host-stepped control (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import to_dev

w = configs.C1_S3E4
u0 = w.initial_condition()
ctx = pkg.Context(0, orth=sys.argv[1] if len(sys.argv) > 1 else None)
op = pkg.Operator(ctx, w.spec())
r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, 5 * w.dt, tol=w.tol, max_basis=30, orth_length=30,
                  use_graph=False)
print(r.steps, r.krylov_iterations)
