"""C1 (sigma = 3e-4 variant, K = 512, N = 4) on the fused cluster engine: us per EPI2 step and the
per-phase SM cycles (expdg_debug_profile), for the controller-latency work."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
w = configs.C1_S3E4
ctx = pkg.Context(0)
op = pkg.Operator(ctx, w.spec())
u0 = torch.tensor(w.initial_condition(), device="cuda:0")
kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
pkg.integrate(ctx, op, u0.clone(), "epi2", w.dt, 20 * w.dt, **kw)  # warm-up
r = pkg.integrate(ctx, op, u0.clone(), "epi2", w.dt, steps * w.dt, **kw)
prof = ctx.debug_profile()
calls = prof.pop("expm_calls")
tot = sum(v for k, v in prof.items() if k != "expm")
us = r.loop_ms * 1e3 / r.steps
print(f"C1s: {r.steps} steps, {us:.1f} us/step, {r.krylov_iterations / r.steps:.2f} Krylov its/step, "
      f"path {ctx.last_path()}")
for k, v in prof.items():
    print(f"  {k:8s} {v / r.steps:10.0f} cycles/step  {100 * v / max(tot, 1):5.1f} %  ~{us * v / max(tot, 1):6.1f} us")
print(f"  expm calls per step {calls / r.steps:.2f}, cycles per call {prof['expm'] / max(calls, 1):.0f}")
xp = ctx.debug_expm_profile()
nc = max(xp["calls"], 1)
print("  expm sub-phases, cycles per call: " + ", ".join(f"{k} {xp[k] / nc:.0f}" for k in
      ("norm_scale", "pade", "lu", "backsub", "squarings")) + f"; squarings per call {xp['squarings_taken'] / nc:.2f}")
