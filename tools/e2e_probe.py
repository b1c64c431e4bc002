"""Host-side cost of one integrate() call on C4: device-resident vs host buffers vs the bare
H2D + D2H of the state (EXPDG_TIMING=1 adds integrate's own phase timings on stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402,F401
import torch  # noqa: E402
import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402
w = configs.C4
u0 = w.initial_condition(); dt = w.time_step(u0)
kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
ctx = pkg.Context(0); op = pkg.Operator(ctx, w.spec())
ud = torch.tensor(u0, device='cuda:0')
for _ in range(2): pkg.integrate(ctx, op, ud, 'epi2', dt, dt, **kw)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3): r = pkg.integrate(ctx, op, ud, 'epi2', dt, dt, **kw)
torch.cuda.synchronize(); t1 = time.perf_counter()
print('device-resident call ms', (t1 - t0) / 3 * 1e3, 'loop_ms', r.loop_ms)
uh = torch.empty(ud.numel(), dtype=torch.float64, pin_memory=True); uh.copy_(ud.cpu())
t0 = time.perf_counter()
for _ in range(3):
    ud.copy_(uh, non_blocking=True); uh.copy_(ud, non_blocking=True); torch.cuda.synchronize()
t1 = time.perf_counter()
print('h2d+d2h ms', (t1 - t0) / 3 * 1e3)
uhn = uh.numpy()
t0 = time.perf_counter()
for _ in range(3): r = pkg.integrate(ctx, op, uhn, 'epi2', dt, dt, **kw)
t1 = time.perf_counter()
print('host call ms', (t1 - t0) / 3 * 1e3, 'loop_ms', r.loop_ms)
