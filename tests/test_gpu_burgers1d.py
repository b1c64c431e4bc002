"""GPU parity: 1D Burgers operator (proj/src/burgers.cpp) vs the CPU oracle."""
import math

import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu

TOL_OP = 1e-13  # fp64 operator application, rounding-order differences only


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


CASES = [
    dict(order=4, nx=64, periodic=True, flux="ef", sigma=1.0, kappa=1e-2),
    dict(order=4, nx=64, periodic=True, flux="lf", sigma=0.0, kappa=1e-2),
    dict(order=7, nx=48, periodic=True, flux="lf", sigma=0.0, kappa=1e-4),
    dict(order=3, nx=9, periodic=False, flux="ef", sigma=1e-3, kappa=0.02),
    dict(order=2, nx=8, periodic=False, flux="lf", sigma=0.0, kappa=0.05),
    dict(order=5, nx=7, periodic=True, flux="ef", sigma=2e-3, kappa=0.04, sigma_adaptive=True),
    dict(order=1, nx=130, periodic=True, flux="ef", sigma=0.3, kappa=0.1),
    dict(order=8, nx=300, periodic=False, flux="lf", sigma=0.0, kappa=0.01),
]


@pytest.mark.parametrize("case", CASES)
def test_apply_linear_nonlinear_full(ctx, case):
    rng = np.random.default_rng(7)
    spec = pkg.OperatorSpec("burgers1d", box=(0.0, 2 * math.pi, 0, 1, 0, 1), **case)
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    ref = rng.standard_normal(op.dim)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    xd = to_dev(x)
    assert rel(to_host(op.apply_linear(xd)), orc.apply_linear(ref, x)) < TOL_OP
    assert rel(to_host(op.apply_nonlinear(xd)), orc.apply_nonlinear(ref, x)) < TOL_OP
    assert rel(to_host(op.full_rhs(xd)), orc.full_rhs(x)) < TOL_OP


def test_linearity_and_splitting_invariance(ctx):
    rng = np.random.default_rng(11)
    spec = pkg.OperatorSpec("burgers1d", 4, 32, box=(0, 1, 0, 1, 0, 1), kappa=0.03, flux="ef", sigma=1e-3)
    op = pkg.Operator(ctx, spec)
    op.linearize(to_dev(rng.standard_normal(op.dim)))
    u, w = to_dev(rng.standard_normal(op.dim)), to_dev(rng.standard_normal(op.dim))
    lhs = to_host(op.apply_linear(1.7 * u - 0.4 * w))
    rhs = 1.7 * to_host(op.apply_linear(u)) - 0.4 * to_host(op.apply_linear(w))
    assert np.linalg.norm(lhs - rhs) / (1 + np.linalg.norm(rhs)) < 1e-12
    r1 = to_host(op.apply_linear(u) + op.apply_nonlinear(u))
    op.linearize(to_dev(rng.standard_normal(op.dim)))
    r2 = to_host(op.apply_linear(u) + op.apply_nonlinear(u))
    assert rel(r1, r2) < 1e-12
    assert rel(to_host(op.full_rhs(u)), r1) < 1e-12


def test_errors_map_to_reference_exceptions(ctx):
    with pytest.raises(ValueError):
        pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", 4, 8, kappa=0.0))
    with pytest.raises(ValueError):
        pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", 4, 8, sigma=-1.0))
    with pytest.raises(pkg.UnsupportedError):
        pkg.Operator(ctx, pkg.OperatorSpec("burgers2d", 4, 8, 8, over_integrate=True))
    op = pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", 4, 8))
    bad = np.zeros(op.dim)
    bad[3] = np.nan
    with pytest.raises(ValueError):
        op.linearize(to_dev(bad))


def test_c1_blows_up_at_the_reference_step(ctx):
    # C1 as specified (sigma = 1 in the explicit N) blows up in the reference algorithm
    # at step 3 (oracle); the device must report the same blow_up_step.
    import oracle
    w = configs.C1
    u0 = w.initial_condition()
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, w.steps * w.dt, tol=w.tol, max_basis=30,
                                             orth_length=30)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, w.steps * w.dt, tol=w.tol, max_basis=30, orth_length=30)
    assert orc.status == "blew_up" and r.status == "blew_up"
    assert r.blow_up_step == orc.blow_up_step == 3


@pytest.mark.parametrize("use_graph", [True, False])
def test_c1_sigma3e4_full_run_parity(ctx, use_graph):
    # Labelled non-degenerate C1 variant (sigma = 3e-4): all 1000 steps.
    w = configs.C1_S3E4
    steps = w.steps if use_graph else 50
    u0 = w.initial_condition()
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, steps * w.dt, tol=w.tol, max_basis=30,
                                             orth_length=30)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, steps * w.dt, tol=w.tol, max_basis=30, orth_length=30,
                      use_graph=use_graph)
    assert r.status == orc.status == "completed" and r.steps == orc.steps == steps
    assert rel(to_host(r.u), orc.u) <= 1e-9  # north-star bar
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1  # Krylov dims per step +-1
    assert abs(r.max_abs - orc.max_abs) <= 1e-9 * orc.max_abs


def test_integrate_host_buffers(ctx):
    w = configs.scaled(configs.C1_S3E4, 64, steps=5)
    u0 = w.initial_condition()
    op = pkg.Operator(ctx, w.spec())
    r_dev = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, w.steps * w.dt, tol=w.tol, max_basis=30,
                          orth_length=30)
    r_host = pkg.integrate(ctx, op, u0.copy(), "epi2", w.dt, w.steps * w.dt, tol=w.tol, max_basis=30,
                           orth_length=30)
    assert np.array_equal(to_host(r_dev.u), r_host.u)  # deterministic reductions: identical bits


def test_step_epi2_matches_oracle(ctx):
    import oracle
    w = configs.scaled(configs.C1_S3E4, 128, steps=1)
    u0 = w.initial_condition()
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, w.dt, tol=1e-12, max_basis=128, orth_length=128)
    op = pkg.Operator(ctx, w.spec())
    u = to_dev(u0)
    op.linearize(u)
    u, st = pkg.step_epi2(ctx, op, u, w.dt, tol=1e-12)
    assert rel(to_host(u), orc.u) < 1e-11
    assert abs(st.iterations - orc.krylov_iterations) <= 1
