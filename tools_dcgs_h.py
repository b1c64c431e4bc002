"""Debug: Hessenberg of one phi call (CGS2 vs DCGS2 selected by EXPDG_ORTH)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle
import paper_2011_01316_b200 as pkg
from tests.gpu_util import to_dev, to_host

u0, src, cfg = oracle.harness_burgers("burgers-smooth", 40, 4, "ef", 3e-4)
ctx = pkg.Context(0)
spec = pkg.OperatorSpec("burgers1d", 4, 40, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                        flux=cfg["flux"], sigma=cfg["sigma"], over_integrate=cfg["over_integrate"])
op = pkg.Operator(ctx, spec)
u = to_dev(u0)
op.linearize(u)
r = op.apply_linear(u) + op.apply_nonlinear(u)
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 16
dt = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
try:
    out, st = pkg.phi_combination(ctx, op, [None, r], dt, tol=1e-12, max_basis=mb, orth_length=mb)
    print("ok", st.iterations, st.substeps)
except Exception as e:
    print("err", e)
H = ctx.debug_hessenberg()
m = int(ctx.debug_state()["mc"])
np.save(f"gpurun_out/H_{os.environ.get('EXPDG_ORTH', 'dcgs2')}.npy", H[:m + 1, :m])
print("mc", m, ctx.debug_state())
