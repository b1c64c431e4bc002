"""GPU: size-independent properties of the bench configs at their FULL sizes (C3 512^2,
C4 1024^2, C5 64^3), where the oracle cannot follow (one C4 step on the CPU is minutes):

* determinism: the reductions are fixed-order (warp -> block -> last-CTA grid sums, no
  fp64 atomics), so two runs of the same steps give the same bits;
* conservation: with periodic boundaries the DG residual and the linearised operator
  conserve every component's integral (1^T M R = 1^T M L x = 0, proj/tests/test_burgers.cpp
  :184-202 and the reference's criterion 11), so every Krylov vector is mass-free and an
  EPI2 step preserves the integrals to rounding, whatever the Krylov tolerance.
"""
import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import to_dev, to_host

pytestmark = pytest.mark.gpu


def integrals(w, q):
    """Per-component integrals sum_e sum_nodes (prod_d w_i h_d / 2) q (uniform meshes)."""
    _, wts, _ = pkg.lgl_basis(w.order)
    dim = {"burgers2d": 2, "euler2d": 2, "euler3d": 3}[w.kind]
    comps = {"burgers2d": 1, "euler2d": 4, "euler3d": 5}[w.kind]
    wn = wts
    for _ in range(dim - 1):
        wn = np.multiply.outer(wn, wts)
    wn = wn.reshape(-1)  # tensor weights, x fastest (products commute)
    q = q.reshape(-1, comps, wn.size)
    vol = 1.0
    for d in range(dim):
        n = (w.nx, w.ny, w.nz)[d]
        vol *= (w.box[2 * d + 1] - w.box[2 * d]) / n / 2.0
    tot = np.einsum("ecn,n->c", q, wn) * vol
    mag = np.einsum("ecn,n->c", np.abs(q), wn) * vol
    return tot, mag


@pytest.mark.parametrize("name,steps", [("C3", 2), ("C4", 1), ("C5", 1)])
def test_full_size_steps_are_deterministic_and_conservative(name, steps):
    w = configs.ALL[name]
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    ctx = pkg.Context(0)
    op = pkg.Operator(ctx, w.spec())
    runs = []
    for _ in range(2):
        r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, steps * dt, **kw)
        assert r.status == "completed" and r.steps == steps
        runs.append((to_host(r.u), list(r.iters_per_step)))
    (ua, ia), (ub, ib) = runs
    assert np.array_equal(ua, ub), "two runs of the same steps differ"
    assert ia == ib
    t0, mag = integrals(w, u0)
    t1, _ = integrals(w, ua)
    scale = np.maximum(mag, 1e-3 * mag.max())  # C5: the w-momentum starts identically zero
    assert np.all(np.abs(t1 - t0) <= 1e-12 * scale), (t1 - t0) / scale
