"""GPU: the device path against the committed golden end states (tests/golden/)."""
import os

import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.golden import make_golden
from tests.gpu_util import rel, to_dev, to_host

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("case", make_golden.CASES, ids=[c[0] for c in make_golden.CASES])
def test_device_matches_golden(case):
    name, cfg, nx, steps, integ = case
    g = np.load(os.path.join(HERE, name + ".npz"))
    w = configs.scaled(configs.ALL[cfg], nx, steps=steps)
    ctx = pkg.Context(0)
    dt = float(g["dt"])
    r = pkg.integrate(ctx, pkg.Operator(ctx, w.spec()), to_dev(g["u0"]), integ, dt, steps * dt, tol=w.tol,
                      max_basis=w.max_basis, orth_length=w.max_basis)
    assert r.status == "completed" and r.steps == steps
    assert rel(to_host(r.u), g["u"]) <= 1e-9
    dd = np.diff(np.concatenate([[0], r.iters_per_step]))
    dg = np.diff(np.concatenate([[0], g["iters"]]))
    assert np.max(np.abs(dd - dg)) <= (2 if integ.startswith("exprb") else 1)
