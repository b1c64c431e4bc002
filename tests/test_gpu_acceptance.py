"""The reference's own acceptance criteria replayed on the DEVICE path.

The device integrates the harness problems of proj/src/harness.cpp:48-142
(over-integrated LDG Burgers on (0,1) with zero Dirichlet data, optional MMS
source) with exactly the reference's settings (proj/tests/acceptance.cpp), and
must reproduce the digits the reference printed in proj/test_output.txt:18-28.
The oracle only supplies initial states / reference solutions / error norms
(checker side).
"""
import math

import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from tests.gpu_util import to_dev, to_host

pytestmark = pytest.mark.gpu

KRYLOV = dict(tol=1e-12, max_basis=128, orth_length=128)  # ExperimentConfig defaults


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def device_problem(ctx, problem, ne, k, flux="", sigma=0.0):
    u0, src, cfg = oracle.harness_burgers(problem, ne, k, flux, sigma)
    spec = pkg.OperatorSpec("burgers1d", k, ne, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                            flux=cfg["flux"], sigma=cfg["sigma"], sigma_adaptive=cfg["sigma_adaptive"],
                            over_integrate=cfg["over_integrate"])
    op = pkg.Operator(ctx, spec)
    if np.any(src != 0.0):
        op.set_source(to_dev(src))
    return op, u0


def test_over_integrated_operator_matches_oracle(ctx):
    rng = np.random.default_rng(3)
    for k in range(1, 9):
        for periodic in (True, False):
            spec = pkg.OperatorSpec("burgers1d", k, 9, box=(0, 1, 0, 1, 0, 1), periodic=periodic, kappa=0.04,
                                    flux="ef", sigma=2e-3, over_integrate=True)
            op = pkg.Operator(ctx, spec)
            orc = oracle.Problem("burgers1d", k, 9, box=(0, 1, 0, 1, 0, 1), periodic=periodic, kappa=0.04,
                                 flux="ef", sigma=2e-3, over_integrate=True)
            ref, x = rng.standard_normal(op.dim), rng.standard_normal(op.dim)
            op.linearize(to_dev(ref))
            for dev_f, orc_f in ((op.apply_linear, lambda v: orc.apply_linear(ref, v)),
                                 (op.apply_nonlinear, lambda v: orc.apply_nonlinear(ref, v)),
                                 (op.full_rhs, orc.full_rhs)):
                a, b = to_host(dev_f(to_dev(x))), orc_f(x)
                assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b), (k, periodic)


def test_criterion_5_large_courant_epi2(ctx):
    # proj/test_output.txt:22 — "Cr_d=161.0, EPI2 completed with max|u| ratio 1.0000"
    op, u0 = device_problem(ctx, "burgers-smooth", 40, 4, "ef", 3e-4)
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", 0.1, 1.0, **KRYLOV)
    assert r.status == "completed" and r.steps == 10
    assert f"{r.max_abs / np.abs(u0).max():.4f}" == "1.0000"


def test_criterion_4_temporal_orders(ctx):
    # proj/test_output.txt:21 — EPI2 orders 1.974 2.044 2.037 (err@0.01 4.942e-06),
    # EXPRB32 orders 2.641 2.881 3.001
    uref = oracle.rk4_reference("burgers-smooth", 40, 4, "lf", 1, 1e-5, 1.0)
    dts = [0.5, 0.25, 0.1, 0.05, 0.01]
    for integ, want in (("epi2", ["1.974", "2.044", "2.037"]), ("exprb32", ["2.641", "2.881", "3.001"])):
        errs = []
        for dt in dts:
            op, u0 = device_problem(ctx, "burgers-smooth", 40, 4, "lf")
            r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, 1.0, **KRYLOV)
            assert r.status == "completed"
            errs.append(oracle.l2_error_discrete("burgers-smooth", 40, 4, to_host(r.u), 40, 4, uref))
        orders = [f"{math.log(errs[i - 1] / errs[i]) / math.log(dts[i - 1] / dts[i]):.3f}" for i in (2, 3, 4)]
        assert orders == want, (integ, orders)
        if integ == "epi2":
            assert f"{errs[4]:.3e}" == "4.942e-06"


@pytest.mark.parametrize("k,flux,errs_want,orders_want", [
    (2, "lf", ["2.455e-06", "3.051e-07", "3.807e-08", "4.755e-09"], ["3.008", "3.003", "3.001"]),
    (4, "lf", None, ["5.003", "5.001", "5.000"]),
    (3, "ef", None, ["3.077", "3.019", "3.005"]),
])
def test_criteria_2_3_manufactured_solution(ctx, k, flux, errs_want, orders_want):
    # proj/test_output.txt:19-20 — exprb32, dt 5e-5, t 0.01, MMS source term on the device
    errs = []
    for ne in (20, 40, 80, 160):
        op, u0 = device_problem(ctx, "burgers-mms", ne, k, flux, 0.0)
        r = pkg.integrate(ctx, op, to_dev(u0), "exprb32", 5e-5, 0.01, **KRYLOV)
        assert r.status == "completed"
        errs.append(oracle.l2_error_exact("burgers-mms", ne, k, to_host(r.u), 0.01))
    if errs_want:
        assert [f"{e:.3e}" for e in errs] == errs_want
    assert [f"{math.log2(errs[i - 1] / errs[i]):.3f}" for i in (1, 2, 3)] == orders_want


def test_criterion_9_burgers_orders(ctx):
    # proj/test_output.txt:26 — "Burgers orders 1.04/2.04/2.88/3.70"
    uref = oracle.rk4_reference("burgers-smooth", 20, 3, "lf", 1, 1e-5, 1.0)
    got = []
    for integ in ("exp_euler", "epi2", "exprb32", "exprb42"):
        e = []
        for dt in (0.1, 0.05):
            op, u0 = device_problem(ctx, "burgers-smooth", 20, 3, "lf")
            r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, 1.0, **KRYLOV)
            e.append(oracle.l2_error_discrete("burgers-smooth", 20, 3, to_host(r.u), 20, 3, uref))
        got.append(f"{math.log(e[0] / e[1]) / math.log(2.0):.2f}")
    assert got == ["1.04", "2.04", "2.88", "3.70"]


@pytest.mark.parametrize("over_integrate", [True, False])
def test_source_function_matches_weak_load(ctx, over_integrate):
    # expdg_op_set_source_fn builds (s, l_j) itself (proj/src/burgers.cpp:80-92)
    u0, src, cfg = oracle.harness_burgers("burgers-mms", 20, 3, "lf", 0.0, over_integrate=over_integrate)
    spec = pkg.OperatorSpec("burgers1d", 3, 20, box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"],
                            flux=cfg["flux"], over_integrate=over_integrate)
    a, b = pkg.Operator(ctx, spec), pkg.Operator(ctx, spec)
    a.set_source(to_dev(src))
    b.set_source_function(lambda x: oracle.mms_source(x, cfg["kappa"]))
    x = to_dev(u0)
    ya, yb = to_host(a.full_rhs(x)), to_host(b.full_rhs(x))
    assert np.linalg.norm(ya - yb) <= 1e-13 * np.linalg.norm(ya)


def test_criterion_8_vortex_orders_roe(ctx):
    # proj/test_output.txt:25 — euler-vortex (harness default flux = Roe), exprb42,
    # ne {256, 1024}, dt 0.01, t 1: k=1 rho order 1.725; k=2 2.709 (err 1.486e-05); k=3 3.781
    want = {1: "1.725", 2: "2.709", 3: "3.781"}
    for k in (1, 2, 3):
        errs = []
        for ne in (256, 1024):
            nx = int(round(math.sqrt(ne)))
            u0 = oracle.harness_u0("euler-vortex", ne, k)
            op = pkg.Operator(ctx, pkg.OperatorSpec("euler2d", k, nx, nx, box=(0.0, 10.0, -5.0, 5.0, 0, 1),
                                                    euler_flux="roe"))
            r = pkg.integrate(ctx, op, to_dev(u0), "exprb42", 0.01, 1.0, **KRYLOV)
            assert r.status == "completed" and r.steps == 100
            errs.append(oracle.l2_error_exact("euler-vortex", ne, k, to_host(r.u), 1.0, 0))
        assert f"{math.log2(errs[0] / errs[1]):.3f}" == want[k]
        if k == 2:
            assert f"{errs[1]:.3e}" == "1.486e-05"


def test_device_run_against_a_stored_reference_file(ctx, tmp_path):
    # the harness's reference-file cache (proj/src/harness.cpp:355-386): an RK4 fine-step
    # reference written in the expdg-reference-v1 format, loaded back, device EPI2 error vs it
    from paper_2011_01316_b200 import refio
    spec = refio.ReferenceSpec("burgers-smooth", "lf", over_integrate=True, kappa=0.03, integrator="rk4", k=3, ne=20,
                               dt=1e-5, t_final=1.0)
    path = str(tmp_path / refio.reference_filename(spec))
    refio.save_reference(path, spec, oracle.rk4_reference("burgers-smooth", 20, 3, "lf", 1, 1e-5, 1.0))
    uref = refio.load_reference(path, spec)
    op, u0 = device_problem(ctx, "burgers-smooth", 20, 3, "lf")
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", 0.05, 1.0, **KRYLOV)
    err = oracle.l2_error_discrete("burgers-smooth", 20, 3, to_host(r.u), 20, 3, uref)
    direct = oracle.l2_error_discrete("burgers-smooth", 20, 3, to_host(r.u), 20, 3,
                                      oracle.rk4_reference("burgers-smooth", 20, 3, "lf", 1, 1e-5, 1.0))
    assert err == direct and 0 < err < 1e-3  # %.17g files round-trip the reference exactly


def test_criterion_6_energy_identity_on_device_residuals(ctx):
    # proj/tests/acceptance.cpp:241-271 (recorded worst 2.12e-13, tolerance 1e-10): the DEVICE
    # residual L u + N u of the over-integrated EF Burgers operator satisfies the discrete energy
    # identity <u, r> + kappa <q, q> + penalty(u) = 0 (q, the penalty and <.,.> from the checker)
    rng = np.random.default_rng(616)
    worst = 0.0
    for k in range(1, 7):
        kw = dict(box=(0.0, 1.0, 0, 1, 0, 1), periodic=True, kappa=0.04, flux="ef", sigma=2e-3, over_integrate=True)
        op = pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", k, 8, **kw))
        orc = oracle.Problem("burgers1d", k, 8, **kw)
        for _ in range(17):
            u = rng.standard_normal(op.dim)
            ud = to_dev(u)
            op.linearize(ud)
            r = to_host(op.apply_linear(ud) + op.apply_nonlinear(ud))
            _, (_, ip_qq, pen, ip_uu) = oracle.burgers_diag(orc, u, u)
            lhs = oracle.burgers_inner(orc, u, r) + 0.04 * ip_qq + pen
            worst = max(worst, abs(lhs) / (1.0 + ip_uu))
    assert worst <= 1e-10


def test_criteria_7_11_splitting_invariance_and_conservation(ctx):
    # proj/tests/acceptance.cpp:275-331, :467-527: L(a) u + N(a) u independent of a (recorded
    # 6.61e-16) and the mass-weighted mean of the periodic RHS vanishing (recorded 1.70e-16)
    rng = np.random.default_rng(707)
    worst_split, worst_cons = 0.0, 0.0
    kw = dict(box=(0.0, 1.0, 0, 1, 0, 1), periodic=True, kappa=0.02, flux="ef", sigma=3e-4)
    op1, op2 = pkg.Operator(ctx, pkg.OperatorSpec("burgers1d", 3, 9, **kw)), pkg.Operator(
        ctx, pkg.OperatorSpec("burgers1d", 3, 9, **kw))
    orc = oracle.Problem("burgers1d", 3, 9, **kw)
    for _ in range(25):
        u, a, b = (rng.standard_normal(op1.dim) for _ in range(3))
        op1.linearize(to_dev(a))
        op2.linearize(to_dev(b))
        ud = to_dev(u)
        r1 = to_host(op1.apply_linear(ud) + op1.apply_nonlinear(ud))
        r2 = to_host(op2.apply_linear(ud) + op2.apply_nonlinear(ud))
        worst_split = max(worst_split, np.linalg.norm(r1 - r2) / np.linalg.norm(r1))
        worst_cons = max(worst_cons, abs(oracle.burgers_inner(orc, np.ones(op1.dim), r1)) /
                         (1.0 + np.linalg.norm(r1)))
    ek = dict(box=(0.0, 10.0, -5.0, 5.0, 0, 1), euler_flux="lf")
    e1 = pkg.Operator(ctx, pkg.OperatorSpec("euler2d", 2, 3, 3, **ek))
    e2 = pkg.Operator(ctx, pkg.OperatorSpec("euler2d", 2, 3, 3, **ek))
    npe = 9
    for _ in range(25):
        def state():
            q = np.empty(9 * 4 * npe)
            for e in range(9):
                blk = q[e * 4 * npe:(e + 1) * 4 * npe].reshape(4, npe)
                rho, vx, vy, p = (rng.uniform(0.5, 2.0, npe), rng.uniform(-1, 1, npe), rng.uniform(-1, 1, npe),
                                  rng.uniform(0.5, 2.0, npe))
                blk[0], blk[1], blk[2], blk[3] = rho, rho * vx, rho * vy, p / 0.4 + 0.5 * rho * (vx * vx + vy * vy)
            return q
        q, a, b = state(), state(), state()
        e1.linearize(to_dev(a))
        e2.linearize(to_dev(b))
        qd = to_dev(q)
        r1 = to_host(e1.apply_linear(qd) + e1.apply_nonlinear(qd))
        r2 = to_host(e2.apply_linear(qd) + e2.apply_nonlinear(qd))
        worst_split = max(worst_split, np.linalg.norm(r1 - r2) / np.linalg.norm(r1))
    assert worst_split <= 1e-12
    assert worst_cons <= 1e-12


def test_criterion_10_exp_euler_joint_estimate(ctx):
    # proj/test_output.txt:27 — exp_euler, k = 2, (ne, dt) = (10, 0.2), (20, 0.1), (40, 0.05)
    # against the RK4 k = 6, ne = 80, dt = 5e-6 reference: errors 8.303e-03 3.847e-03 1.866e-03
    uref = oracle.rk4_reference("burgers-smooth", 80, 6, "lf", 1, 5e-6, 1.0)
    errs = []
    for ne, dt in ((10, 0.2), (20, 0.1), (40, 0.05)):
        op, u0 = device_problem(ctx, "burgers-smooth", ne, 2, "lf")
        r = pkg.integrate(ctx, op, to_dev(u0), "exp_euler", dt, 1.0, **KRYLOV)
        assert r.status == "completed"
        errs.append(oracle.l2_error_discrete("burgers-smooth", ne, 2, to_host(r.u), 80, 6, uref))
    assert [f"{e:.3e}" for e in errs] == ["8.303e-03", "3.847e-03", "1.866e-03"]
