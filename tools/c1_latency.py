"""C1 (labelled sigma = 3e-4 variant) step latency on the device vs the oracle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import to_dev

w = configs.C1_S3E4
u0 = w.initial_condition()
ctx = pkg.Context(0, orth=sys.argv[1] if len(sys.argv) > 1 else None)
op = pkg.Operator(ctx, w.spec())
kw = dict(tol=w.tol, max_basis=30, orth_length=30)
pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, 20 * w.dt, **kw)
r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, w.steps * w.dt, **kw)
print(f"device: {r.loop_ms / r.steps * 1e3:.1f} us/step, {r.krylov_iterations / r.steps:.1f} iters/step, "
      f"launches {ctx.kernel_launches}")
prof = ctx.debug_profile()
print("fused phases (us/step at 1.9 GHz):", {k: round(v / 1.9e3 / r.steps, 1) for k, v in prof.items()})
if len(sys.argv) > 2:
    import oracle
    from tests.gpu_util import oracle_problem
    t = time.perf_counter()
    o = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, w.steps * w.dt, **kw)
    print(f"oracle: {(time.perf_counter() - t) / o.steps * 1e6:.1f} us/step")
