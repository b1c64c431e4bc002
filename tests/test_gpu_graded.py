"""GPU parity on graded meshes: build_quad_mesh's grading lists (proj/src/mesh.cpp:96-120)
through expdg_op_desc.grade_x / grade_y (/ grade_z for the 3D extension), against the oracle
built on the same breakpoints."""
import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host
from tests.test_gpu_euler2d import random_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def graded(a, b, n, ratio):
    """Geometric grading a..b with h_{i+1} / h_i = ratio, exact end points."""
    w = ratio ** np.arange(n)
    xs = a + (b - a) * np.concatenate([[0.0], np.cumsum(w) / w.sum()])
    xs[0], xs[-1] = a, b
    return xs


@pytest.mark.parametrize("flux", ["lf", "roe"])
@pytest.mark.parametrize("order,nx,ny", [(2, 5, 4), (4, 9, 7), (4, 33, 3)])
def test_graded_euler2d_operator_matches_oracle(ctx, flux, order, nx, ny):
    rng = np.random.default_rng(order * 31 + nx)
    spec = pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 10, -5, 5, 0, 1), euler_flux=flux,
                            grade_x=graded(0, 10, nx, 1.15), grade_y=graded(-5, 5, ny, 0.8))
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    npe = (order + 1) ** 2
    ref = random_state(rng, nx * ny, npe)
    q = random_state(rng, nx * ny, npe)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < 1e-13
    assert rel(to_host(op.apply_nonlinear(to_dev(q))), orc.apply_nonlinear(ref, q)) < 1e-13
    assert rel(to_host(op.full_rhs(to_dev(q))), orc.full_rhs(q)) < 1e-12
    # grading really changes the operator
    uni = pkg.Operator(ctx, pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 10, -5, 5, 0, 1), euler_flux=flux))
    uni.linearize(to_dev(ref))
    assert rel(to_host(uni.apply_linear(to_dev(x))), to_host(op.apply_linear(to_dev(x)))) > 1e-3


def test_graded_vortex_epi2_matches_oracle(ctx):
    # the C4 vortex on a graded 24^2 mesh (the paper's nonuniform-mesh vortex runs), EPI2 at Cr_a 5
    w = configs.scaled(configs.C4, 24, steps=3)
    spec = w.spec()
    spec.grade_x = graded(0, 10, 24, 1.04)
    spec.grade_y = graded(0, 10, 24, 0.97)
    u0 = w.initial_condition()
    dt = 0.5 * w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    orc = oracle_problem(spec).integrate("epi2", u0, dt, 3 * dt, **kw)
    op = pkg.Operator(ctx, spec)
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, 3 * dt, **kw)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1


def test_graded_euler3d_and_burgers2d_match_oracle(ctx):
    rng = np.random.default_rng(9)
    spec = pkg.OperatorSpec("euler3d", 2, 4, 3, 4, box=(0, 1, 0, 2, 0, 1), grade_x=graded(0, 1, 4, 1.3),
                            grade_y=graded(0, 2, 3, 0.7), grade_z=graded(0, 1, 4, 1.1))
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    npe = 27
    ref = np.empty(48 * 5 * npe)
    for e in range(48):
        blk = ref[e * 5 * npe:(e + 1) * 5 * npe].reshape(5, npe)
        rho, u, v, ww, p = (rng.uniform(0.5, 2, npe), rng.uniform(-1, 1, npe), rng.uniform(-1, 1, npe),
                            rng.uniform(-1, 1, npe), rng.uniform(0.5, 2, npe))
        blk[:] = [rho, rho * u, rho * v, rho * ww, p / 0.4 + 0.5 * rho * (u * u + v * v + ww * ww)]
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < 1e-13
    spec2 = pkg.OperatorSpec("burgers2d", 3, 6, 5, box=(0, 1, 0, 1, 0, 1), kappa=1e-2, flux="lf",
                             grade_x=graded(0, 1, 6, 1.2), grade_y=graded(0, 1, 5, 0.85))
    op2 = pkg.Operator(ctx, spec2)
    orc2 = oracle_problem(spec2)
    ref2 = rng.standard_normal(op2.dim)
    x2 = rng.standard_normal(op2.dim)
    op2.linearize(to_dev(ref2))
    assert rel(to_host(op2.apply_linear(to_dev(x2))), orc2.apply_linear(ref2, x2)) < 1e-13
    assert rel(to_host(op2.full_rhs(to_dev(x2))), orc2.full_rhs(x2)) < 1e-12


def test_bad_grading_lists_are_invalid(ctx):
    # proj/src/mesh.cpp:18-24
    base = dict(box=(0, 1, 0, 1, 0, 1))
    bad_span = np.array([0.0, 0.5, 0.9])
    with pytest.raises(ValueError, match="span"):
        pkg.Operator(ctx, pkg.OperatorSpec("euler2d", 2, 2, 2, grade_x=bad_span, **base))
    with pytest.raises(ValueError, match="increasing"):
        pkg.Operator(ctx, pkg.OperatorSpec("euler2d", 2, 2, 2, grade_y=np.array([0.0, 1.2, 1.0]), **base))
    with pytest.raises(pkg.UnsupportedError):
        pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", 2, 2, grade_x=np.array([0.0, 0.3, 1.0]), **base))


def test_graded_partitioned_matches_single_rank():
    from tests.test_gpu_multirank import run_ranks
    w = configs.scaled(configs.C4, 6, steps=1)
    spec = w.spec()
    spec.grade_x = graded(0, 10, 6, 1.2)
    spec.grade_y = graded(0, 10, 6, 0.8)
    rng = np.random.default_rng(2)
    ref = w.initial_condition()
    x = rng.standard_normal(ref.size)
    ctx = pkg.Context(0)
    whole = pkg.Operator(ctx, spec)
    whole.linearize(to_dev(ref))
    y_whole = to_host(whole.apply_linear(to_dev(x)))
    blk = spec.nx * 25 * 4
    rows = [(0, 3), (3, 6)]

    def fn(r, c):
        import copy
        s = copy.copy(spec)
        s.part = rows[r]
        op = pkg.Operator(c, s)
        sl = slice(rows[r][0] * blk, rows[r][1] * blk)
        op.linearize(to_dev(ref[sl]))
        return to_host(op.apply_linear(to_dev(x[sl])))

    out = run_ranks(2, fn)
    assert np.array_equal(np.concatenate(out), y_whole)
