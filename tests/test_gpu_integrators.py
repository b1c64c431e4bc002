"""GPU parity of the device time loop beyond EPI2: exp_euler (operator frozen at
u0, proj/src/integrators.cpp:67-74, :150), IOP windows on a DG operator
(proj/src/phi.cpp:91-93, :171-177), and the full-size C2 outcome (the reference
algorithm fails its 40-substep budget at step 1: KrylovError -> blew_up)."""
import math

import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def _dims(r):
    return np.diff(np.concatenate([[0], r.iters_per_step]))


@pytest.mark.parametrize("kind", ["burgers1d", "euler2d"])
def test_exp_euler_matches_oracle(ctx, kind):
    if kind == "burgers1d":
        w = configs.scaled(configs.C1_S3E4, 64, steps=5)
        dt = w.dt
    else:
        w = configs.scaled(configs.C4, 12, steps=3)
    u0 = w.initial_condition()
    dt = w.time_step(u0) if w.dt is None else w.dt
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    orc = oracle_problem(w.spec()).integrate("exp_euler", u0, dt, w.steps * dt, **kw)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "exp_euler", dt, w.steps * dt, **kw)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    assert np.max(np.abs(_dims(r) - _dims(orc))) <= 1


def test_iop_window_on_dg_operator(ctx):
    # incomplete orthogonalisation (orth_length < max_basis) on the C4 operator
    w = configs.scaled(configs.C4, 12, steps=2)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=40, orth_length=6)
    orc = oracle_problem(w.spec()).integrate("epi2", u0, dt, w.steps * dt, **kw)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, w.steps * dt, **kw)
    assert r.status == orc.status
    if r.status == "completed":
        assert rel(to_host(r.u), orc.u) <= 1e-9
        assert np.max(np.abs(_dims(r) - _dims(orc))) <= 1


def test_c2_full_size_fails_like_the_reference(ctx):
    # C2 at full size (K = 2^20, N = 7, 8.4M DOF): KrylovError (substep budget) at step 1;
    # the oracle shows the same outcome at K = 2^12, 2^14 with the same Courant numbers.
    w = configs.C2
    u0 = w.initial_condition()
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, 3 * w.dt, tol=w.tol, max_basis=30, orth_length=30)
    assert r.status == "blew_up" and r.blow_up_step == 1
    assert r.krylov_iterations == 0  # the failed call's statistics are dropped, as in the reference
    small = configs.scaled(w, 1 << 12)
    kap = 1e-4 * 256
    spec = pkg.OperatorSpec("burgers1d", 7, 1 << 12, box=(0, 2 * math.pi, 0, 1, 0, 1), kappa=kap, flux="lf")
    orc = oracle_problem(spec).integrate("epi2", small.initial_condition(), 1e-4 * 256, 2 * 1e-4 * 256, tol=1e-10,
                                         max_basis=30, orth_length=30)
    assert orc.status == "blew_up" and orc.blow_up_step == 1


def test_step_epi2_euler_matches_one_step_integrate(ctx):
    w = configs.scaled(configs.C4, 8, steps=1)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, dt, tol=w.tol, max_basis=40, orth_length=40)
    u = to_dev(u0)
    op.linearize(u)
    u, st = pkg.step_epi2(ctx, op, u, dt, tol=w.tol, max_basis=40, orth_length=40)
    assert rel(to_host(u), to_host(r.u)) < 1e-12
    assert st.iterations == r.krylov_iterations


@pytest.mark.parametrize("integ", ["exprb32", "exprb42"])
@pytest.mark.parametrize("kind", ["burgers1d", "euler2d"])
def test_exprb_matches_oracle(ctx, kind, integ):
    # proj/src/integrators.cpp:85-113: two phi calls per step (p = 1 then p = 3)
    if kind == "burgers1d":
        w = configs.scaled(configs.C1_S3E4, 64, steps=4)
    else:
        w = configs.scaled(configs.C4, 10, steps=2)
    u0 = w.initial_condition()
    dt = w.time_step(u0) if w.dt is None else w.dt
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    orc = oracle_problem(w.spec()).integrate(integ, u0, dt, w.steps * dt, **kw)
    op = pkg.Operator(ctx, w.spec())
    for use_graph in (True, False):
        r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, w.steps * dt, use_graph=use_graph, **kw)
        assert r.status == orc.status == "completed"
        assert rel(to_host(r.u), orc.u) <= 1e-9
        assert np.max(np.abs(_dims(r) - _dims(orc))) <= 2  # two phi calls per step, +-1 each
