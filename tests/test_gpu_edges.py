"""GPU edge cases of the device path against the oracle: single-element periodic
meshes (an element is its own neighbour), a final step shorter than dt (the dt
sequence of proj/src/integrators.cpp:155-157), p = 0 (a plain exponential), a
Krylov space as large as the problem, all-zero and non-finite inputs, the
highest device orders, and partitioned ranks owning a single layer."""
import math

import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


@pytest.mark.parametrize("kind,order,nx,ny", [("burgers1d", 3, 1, 1), ("burgers1d", 8, 2, 1), ("euler2d", 2, 1, 1),
                                              ("euler2d", 8, 1, 2), ("burgers2d", 4, 1, 1)])
def test_tiny_periodic_meshes(ctx, kind, order, nx, ny):
    rng = np.random.default_rng(order * 10 + nx)
    kw = dict(box=(0.0, 2.0, 0.0, 2.0, 0, 1), periodic=True)
    if kind == "euler2d":
        kw["euler_flux"] = "lf"
    else:
        kw.update(kappa=0.05, flux="ef", sigma=1e-3)
    spec = pkg.OperatorSpec(kind, order, nx, ny, **kw)
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    if kind == "euler2d":
        npe = (order + 1) ** 2
        ref = np.concatenate([np.concatenate([np.full(npe, 1.2), np.full(npe, 0.1), np.full(npe, -0.2),
                                              np.full(npe, 3.0)]) + 0.01 * rng.standard_normal(4 * npe)
                              for _ in range(nx * ny)])
    else:
        ref = rng.standard_normal(op.dim)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < 1e-13
    assert rel(to_host(op.full_rhs(to_dev(ref))), orc.full_rhs(ref)) < 1e-12


def test_short_last_step_matches_oracle(ctx):
    # t_final = 3.5 dt: three full steps and a half step
    w = configs.scaled(configs.C1_S3E4, 48, steps=1)
    u0 = w.initial_condition()
    kw = dict(tol=w.tol, max_basis=30, orth_length=30)
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, 3.5 * w.dt, **kw)
    r = pkg.integrate(ctx, pkg.Operator(ctx, w.spec()), to_dev(u0), "epi2", w.dt, 3.5 * w.dt, **kw)
    assert r.steps == orc.steps == 4
    assert abs(r.t - 3.5 * w.dt) < 1e-15 and rel(to_host(r.u), orc.u) < 1e-10


@pytest.mark.parametrize("n", [3, 12, 40])
def test_p0_exponential_and_full_size_krylov(ctx, n):
    # phi_combination with only b_0: exp(dt A) b_0; max_basis >= n + p (breakdown at full size)
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) / math.sqrt(n) - 0.5 * np.eye(n)
    b0 = rng.standard_normal(n)
    op = pkg.Operator(ctx, dense=a)
    out, st = pkg.phi_combination(ctx, op, [to_dev(b0)], 0.7, tol=1e-12, max_basis=128, orth_length=128)
    want = oracle.expm(0.7 * a) @ b0
    assert rel(to_host(out), want) < 1e-10


def test_zero_state_and_nonfinite_input(ctx):
    w = configs.scaled(configs.C1_S3E4, 16, steps=2)
    spec = w.spec()
    op = pkg.Operator(ctx, spec)
    zero = np.zeros(op.dim)
    r = pkg.integrate(ctx, op, to_dev(zero), "epi2", w.dt, 2 * w.dt, tol=w.tol, max_basis=30, orth_length=30)
    assert r.status == "completed" and r.krylov_iterations == 0 and np.all(to_host(r.u) == 0.0)
    # a non-finite Burgers state: the first linearisation throws invalid_argument out of
    # integrate in the reference (proj/src/burgers.cpp:34-35)
    bad = w.initial_condition()
    bad[5] = np.nan
    with pytest.raises(ValueError):
        oracle_problem(spec).integrate("epi2", bad, w.dt, 2 * w.dt, tol=w.tol, max_basis=30, orth_length=30)
    with pytest.raises(ValueError):
        pkg.integrate(ctx, op, to_dev(bad), "epi2", w.dt, 2 * w.dt, tol=w.tol, max_basis=30, orth_length=30)
    # a non-finite Euler state: domain_error at the first linearisation -> blew_up at step 1
    we = configs.scaled(configs.C4, 6, steps=2)
    q = we.initial_condition()
    dt = we.time_step(q)
    q[7] = np.nan
    orc = oracle_problem(we.spec()).integrate("epi2", q, dt, 2 * dt, tol=we.tol, max_basis=40, orth_length=40)
    r = pkg.integrate(ctx, pkg.Operator(ctx, we.spec()), to_dev(q), "epi2", dt, 2 * dt, tol=we.tol, max_basis=40,
                      orth_length=40)
    assert r.status == orc.status == "blew_up" and r.blow_up_step == orc.blow_up_step == 1


def test_single_layer_ranks():
    # every rank owns exactly one element row (the halo is the whole neighbouring slab)
    from tests.test_gpu_multirank import run_ranks
    w = configs.scaled(configs.C4, 4, steps=2)
    spec = w.spec()
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    ctx = pkg.Context(0)
    single = pkg.integrate(ctx, pkg.Operator(ctx, spec), to_dev(u0), "epi2", dt, w.steps * dt, **kw)
    row = spec.nx * (spec.order + 1) ** 2 * 4

    def fn(r, c):
        o = pkg.Operator(c, pkg.OperatorSpec(**{**spec.__dict__, "part": (r, r + 1)}))
        res = pkg.integrate(c, o, to_dev(u0[r * row:(r + 1) * row]), "epi2", dt, w.steps * dt, **kw)
        return to_host(res.u)

    got = run_ranks(spec.ny, fn)
    assert rel(np.concatenate(got), to_host(single.u)) <= 1e-11
