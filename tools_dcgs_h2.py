"""Debug: device Hessenberg (CGS2 / DCGS2) vs the oracle's MGS2 Arnoldi on the dense augmented operator."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle
import paper_2011_01316_b200 as pkg
from tests.gpu_util import to_dev, to_host

u0, src, cfg = oracle.harness_burgers("burgers-smooth", 40, 4, "ef", 3e-4)
dt = float(sys.argv[1]); mb = int(sys.argv[2])
spec = pkg.OperatorSpec("burgers1d", 4, 40, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                        flux=cfg["flux"], sigma=cfg["sigma"], over_integrate=cfg["over_integrate"])
orc = oracle.Problem("burgers1d", 4, 40, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                     flux=cfg["flux"], sigma=cfg["sigma"], over_integrate=cfg["over_integrate"])
n = u0.size
L = np.stack([orc.apply_linear(u0, np.eye(n)[i]) for i in range(n)], axis=1)
r = orc.apply_linear(u0, u0) + orc.apply_nonlinear(u0, u0)
Aug = np.zeros((n + 1, n + 1)); Aug[:n, :n] = dt * L; Aug[:n, n] = dt * r
seed = np.zeros(n + 1); seed[n] = 1.0
_, Href, k, inv, _ = oracle.krylov_build(Aug, seed, mb, mb)
res = {"ref": Href}
for mode in ("cgs2", "dcgs2"):
    os.environ["EXPDG_ORTH"] = mode
    ctx = pkg.Context(0)
    op = pkg.Operator(ctx, spec)
    u = to_dev(u0); op.linearize(u)
    rr = to_dev(r)
    try:
        out, st = pkg.phi_combination(ctx, op, [None, rr], dt, tol=1e-12, max_basis=mb, orth_length=mb, max_substeps=1)
    except Exception as e:
        print(mode, "->", e)
    d = ctx.debug_state()
    print(mode, d)
    H = ctx.debug_hessenberg()[:mb + 1, :mb]
    res[mode] = H
    ctx.close()
print("ref col0", Href[:3, 0], "dcgs col0", res["dcgs2"][:3, 0], "cgs col0", res["cgs2"][:3, 0])
for mode in ("cgs2", "dcgs2"):
    D = np.abs(res[mode] - Href)
    print(mode, "max |H - Href| / max|Href| =", D.max() / np.abs(Href).max(), " per column:",
          " ".join(f"{x:.0e}" for x in D.max(axis=0) / np.abs(Href).max()))
