"""Diagnostics: device DCGS2 Hessenberg (pipelined or two-pass) vs the oracle's MGS2 on the
stiff criterion-5 operator, per basis size (tests/test_gpu_dcgs.py::test_hessenberg_matches_mgs2)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2011_01316_b200 as pkg  # noqa: E402
from tests.gpu_util import to_dev  # noqa: E402
from tests.test_gpu_dcgs import stiff_problem  # noqa: E402

dt = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
ib = int(sys.argv[2]) if len(sys.argv) > 2 else 16  # initial basis (= m: no grows)
u0, spec, orc = stiff_problem()
n = u0.size
L = np.stack([orc.apply_linear(u0, np.eye(n)[i]) for i in range(n)], axis=1)
r = orc.apply_linear(u0, u0) + orc.apply_nonlinear(u0, u0)
aug = np.zeros((n + 1, n + 1))
aug[:n, :n] = dt * L
aug[:n, n] = dt * r
seed = np.zeros(n + 1)
seed[n] = 1.0
for m in (16, 40, 80, 128):
    _, href, _, _, _ = oracle.krylov_build(aug, seed, m, m)
    row = [m]
    for pipe in (False, True):
        ctx = pkg.Context(0, orth="dcgs2", pipelined=pipe)
        op = pkg.Operator(ctx, spec)
        op.linearize(to_dev(u0))
        try:
            pkg.phi_combination(ctx, op, [None, to_dev(r)], dt, tol=1e-12, max_basis=m, orth_length=m, max_substeps=1,
                                initial_basis=m if ib <= 0 else ib)
        except pkg.KrylovError:
            pass
        h = ctx.debug_hessenberg()[:m + 1, :m]
        e = np.abs(h - href)
        row.append(e.max() / np.abs(href).max())
        cols = [float(e[:k + 1, :k].max() / np.abs(href).max()) for k in (8, 16, 24, 32, 48, 64, 96, 128) if k <= m]
        row.append(["%.1e" % c for c in cols])
    print(row, flush=True)
