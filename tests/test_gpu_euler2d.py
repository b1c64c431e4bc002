"""GPU parity: 2D Euler split operator, Lax-Friedrichs and Roe fluxes (proj/src/euler.cpp), vs the oracle."""
import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL_OP = 1e-13


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def random_state(rng, ne, np_):
    q = np.empty(ne * 4 * np_)
    for e in range(ne):
        rho = rng.uniform(0.5, 2.0, np_)
        u = rng.uniform(-1, 1, np_)
        v = rng.uniform(-1, 1, np_)
        p = rng.uniform(0.5, 2.0, np_)
        blk = q[e * 4 * np_:(e + 1) * 4 * np_].reshape(4, np_)
        blk[0], blk[1], blk[2] = rho, rho * u, rho * v
        blk[3] = p / 0.4 + 0.5 * rho * (u * u + v * v)
    return q


@pytest.mark.parametrize("flux", ["lf", "roe"])
@pytest.mark.parametrize("order,nx,ny,box", [
    (1, 3, 3, (0, 10, -5, 5, 0, 1)),
    (2, 4, 3, (0, 10, -5, 5, 0, 1)),
    (3, 5, 7, (0, 1, 0, 2, 0, 1)),
    (4, 8, 8, (0, 10, 0, 10, 0, 1)),
    (4, 33, 2, (0, 10, 0, 10, 0, 1)),
    (7, 3, 4, (0, 3, 1, 2, 0, 1)),
])
def test_apply_matches_oracle(ctx, order, nx, ny, box, flux):
    rng = np.random.default_rng(order * 100 + nx)
    spec = pkg.OperatorSpec("euler2d", order, nx, ny, box=box, euler_flux=flux)
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    npe = (order + 1) ** 2
    ref = random_state(rng, nx * ny, npe)
    q = random_state(rng, nx * ny, npe)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < TOL_OP
    assert rel(to_host(op.apply_nonlinear(to_dev(q))), orc.apply_nonlinear(ref, q)) < TOL_OP
    assert rel(to_host(op.full_rhs(to_dev(q))), orc.full_rhs(q)) < 1e-12


@pytest.mark.parametrize("flux", ["lf", "roe"])
def test_uniform_flow_is_steady(ctx, flux):
    # proj/tests/test_euler.cpp:225-239
    spec = pkg.OperatorSpec("euler2d", 2, 4, 4, box=(0, 10, -5, 5, 0, 1), euler_flux=flux)
    op = pkg.Operator(ctx, spec)
    mean = np.array([1.0, 0.2, 0.0, 1.0 / 0.4 + 0.5 * 0.04])
    q = np.concatenate([np.repeat(mean[c], 9) for c in range(4)] * 16)
    qd = to_dev(q)
    op.linearize(qd)
    assert np.abs(to_host(op.apply_linear(qd) + op.apply_nonlinear(qd))).max() < 1e-12


def test_inadmissible_reference_is_domain_error(ctx):
    spec = pkg.OperatorSpec("euler2d", 2, 2, 2, box=(0, 1, 0, 1, 0, 1), euler_flux="lf")
    op = pkg.Operator(ctx, spec)
    q = random_state(np.random.default_rng(1), 4, 9)
    q[0] = -1.0
    with pytest.raises(ArithmeticError):
        op.linearize(to_dev(q))
    with pytest.raises(pkg.UnsupportedError):
        pkg.Operator(ctx, pkg.OperatorSpec("euler3d", 2, 2, 2, 2, euler_flux="roe"))


@pytest.mark.parametrize("nx", [16, 32])
def test_c4_reduced_mesh_epi2_parity(ctx, nx):
    # C4 physics (strength-5 vortex, LF, Cr_a = 5, tol 1e-10, max dim 40) on a reduced mesh
    w = configs.scaled(configs.C4, nx, steps=3)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    orc = oracle_problem(w.spec()).integrate("epi2", u0, dt, w.steps * dt, tol=w.tol, max_basis=w.max_basis,
                                             orth_length=w.max_basis)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, w.steps * dt, tol=w.tol, max_basis=w.max_basis,
                      orth_length=w.max_basis)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1


def test_inadmissible_state_blows_up_like_reference(ctx):
    # integrate converts the domain_error of linearize into blew_up at step 1
    spec = pkg.OperatorSpec("euler2d", 2, 3, 3, box=(0, 1, 0, 1, 0, 1), euler_flux="lf")
    op = pkg.Operator(ctx, spec)
    q = random_state(np.random.default_rng(2), 9, 9)
    q[5] = -0.5
    r = pkg.integrate(ctx, op, to_dev(q), "epi2", 0.01, 0.05, tol=1e-10, max_basis=20, orth_length=20)
    orc = oracle_problem(spec).integrate("epi2", q, 0.01, 0.05, tol=1e-10, max_basis=20, orth_length=20)
    assert r.status == orc.status == "blew_up" and r.blow_up_step == orc.blow_up_step == 1


@pytest.mark.parametrize("integ", ["epi2", "exprb42"])
def test_roe_vortex_parity(ctx, integ):
    # the harness default flux (EulerConfig{} = Roe, proj/src/harness.cpp:62-66) on the
    # strength-5 C4 vortex, reduced mesh
    w = configs.scaled(configs.C4, 12, steps=3)
    spec = w.spec()
    spec.euler_flux = "roe"
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    orc = oracle_problem(spec).integrate(integ, u0, dt, w.steps * dt, **kw)
    op = pkg.Operator(ctx, spec)
    r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, w.steps * dt, **kw)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1, (d_dev, d_orc)


@pytest.mark.parametrize("gamma", [1.3, 1.67])
def test_gamma_reaches_operator_and_admissibility(ctx, gamma):
    # EulerConfig::gamma (proj/include/expdg/euler.hpp:33-37) in the JVP and in linearize's
    # admissible(q, cfg.gamma) (proj/src/euler.cpp:8-13, :210)
    rng = np.random.default_rng(int(gamma * 100))
    spec = pkg.OperatorSpec("euler2d", 3, 4, 3, box=(0, 1, 0, 1, 0, 1), euler_flux="lf", gamma=gamma)
    op = pkg.Operator(ctx, spec)
    ref = random_state(rng, 12, 16)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), oracle_problem(spec).apply_linear(ref, x)) < TOL_OP


def test_gamma_one_is_inadmissible_like_reference(ctx):
    # gamma = 1: the reference's pressure (gamma - 1)(E - |m|^2 / 2 rho) is identically 0,
    # so admissible() fails and linearize throws domain_error
    spec = pkg.OperatorSpec("euler2d", 2, 2, 2, box=(0, 1, 0, 1, 0, 1), euler_flux="lf", gamma=1.0)
    op = pkg.Operator(ctx, spec)
    ref = random_state(np.random.default_rng(3), 4, 9)
    with pytest.raises(ArithmeticError):
        op.linearize(to_dev(ref))
    with pytest.raises(ArithmeticError):
        oracle_problem(spec).apply_linear(ref, ref)


def test_degenerate_box_is_invalid(ctx):
    # build_quad_mesh: "degenerate box" (proj/src/mesh.cpp:99)
    with pytest.raises(ValueError):
        pkg.Operator(ctx, pkg.OperatorSpec("euler2d", 2, 2, 2, box=(0, 1, 1, 1, 0, 1)))
    with pytest.raises(ValueError):
        pkg.Operator(ctx, pkg.OperatorSpec("euler3d", 2, 2, 2, 2, box=(0, 1, 0, 1, 2, 1)))
