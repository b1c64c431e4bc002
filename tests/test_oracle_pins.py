"""Pins the CPU oracle (oracle/) against the reference's own known answers.

The reference cannot be built here (Eigen3/doctest/CLI11 absent), so the oracle
is pinned by (1) the closed-form assertions of proj/tests/*.cpp restated on the
oracle and (2) the digits recorded by the reference acceptance run,
proj/test_output.txt:18-28, reproduced to every printed digit.
"""
import math

import numpy as np
import pytest

import oracle


def _rng(seed):
    return np.random.default_rng(seed)


# ------------------------------------------------------------------ acceptance digits
def test_acceptance_criterion_5_large_courant():
    # proj/test_output.txt:22 — "Cr_d=161.0, EPI2 completed with max|u| ratio 1.0000;
    # RK2 blew up at step 18"
    import ctypes as C
    out = np.zeros(5)
    oracle.lib().oracle_acc_large_courant(out.ctypes.data_as(C.POINTER(C.c_double)))
    assert f"{out[0]:.1f}" == "161.0"
    assert out[1] == 1.0
    assert f"{out[2]:.4f}" == "1.0000"
    assert out[3] == 1.0 and int(out[4]) == 18


def test_acceptance_criterion_9_ode_orders():
    # proj/test_output.txt:26 — "ODE orders 1.09/2.18/3.06/4.16"
    got = [f"{oracle.lib().oracle_acc_ode_order(k):.2f}" for k in range(4)]
    assert got == ["1.09", "2.18", "3.06", "4.16"]


def test_acceptance_criterion_2_3_mms_digits():
    # proj/test_output.txt:19-20
    import ctypes as C
    e = np.zeros(4)
    P = e.ctypes.data_as(C.POINTER(C.c_double))
    oracle.lib().oracle_acc_mms(2, 0, 0.0, P)
    assert [f"{v:.3e}" for v in e] == ["2.455e-06", "3.051e-07", "3.807e-08", "4.755e-09"]
    assert [f"{math.log2(e[i - 1] / e[i]):.3f}" for i in (1, 2, 3)] == ["3.008", "3.003", "3.001"]
    oracle.lib().oracle_acc_mms(4, 0, 0.0, P)
    assert [f"{math.log2(e[i - 1] / e[i]):.3f}" for i in (1, 2, 3)] == ["5.003", "5.001", "5.000"]
    oracle.lib().oracle_acc_mms(3, 1, 0.0, P)
    assert [f"{math.log2(e[i - 1] / e[i]):.3f}" for i in (1, 2, 3)] == ["3.077", "3.019", "3.005"]


def test_acceptance_criterion_4_temporal_digits():
    # proj/test_output.txt:21 — EPI2 orders 1.974 2.044 2.037 (err@0.01 4.942e-06),
    # EXPRB32 orders 2.641 2.881 3.001
    import ctypes as C
    dts = [0.5, 0.25, 0.1, 0.05, 0.01]
    e = np.zeros(5)
    P = e.ctypes.data_as(C.POINTER(C.c_double))
    orders = lambda: [f"{math.log(e[i - 1] / e[i]) / math.log(dts[i - 1] / dts[i]):.3f}" for i in (2, 3, 4)]
    oracle.lib().oracle_acc_temporal(1, P)
    assert orders() == ["1.974", "2.044", "2.037"]
    assert f"{e[4]:.3e}" == "4.942e-06"
    oracle.lib().oracle_acc_temporal(2, P)
    assert orders() == ["2.641", "2.881", "3.001"]


def test_acceptance_criterion_9_burgers_orders():
    # proj/test_output.txt:26 — "Burgers orders 1.04/2.04/2.88/3.70"
    got = [f"{oracle.lib().oracle_acc_burgers_order(k):.2f}" for k in range(4)]
    assert got == ["1.04", "2.04", "2.88", "3.70"]


@pytest.mark.slow
def test_acceptance_criterion_10_exp_euler_joint():
    # proj/test_output.txt:27 — "errors 8.303e-03 3.847e-03 1.866e-03"
    import ctypes as C
    e = np.zeros(3)
    oracle.lib().oracle_acc_exp_euler_joint(e.ctypes.data_as(C.POINTER(C.c_double)))
    assert [f"{v:.3e}" for v in e] == ["8.303e-03", "3.847e-03", "1.866e-03"]


@pytest.mark.slow
def test_acceptance_criterion_8_vortex_orders():
    # proj/test_output.txt:25 — k=1 rho order 1.725; k=2 2.709 (err 1.486e-05); k=3 3.781
    import ctypes as C
    e = np.zeros(2)
    P = e.ctypes.data_as(C.POINTER(C.c_double))
    want = {1: "1.725", 2: "2.709", 3: "3.781"}
    for k in (1, 2, 3):
        oracle.lib().oracle_acc_vortex(k, P)
        assert f"{math.log2(e[0] / e[1]):.3f}" == want[k]
        if k == 2:
            assert f"{e[1]:.3e}" == "1.486e-05"


# ------------------------------------------------------------------ proj/tests/test_basis.cpp
def test_lgl_low_orders():
    x, w, _ = oracle.lgl(1)
    assert np.allclose(x, [-1, 1]) and np.allclose(w, [1, 1])
    x, w, _ = oracle.lgl(2)
    assert abs(x[1]) <= 1e-15 and abs(w[0] - 1 / 3) < 1e-14 and abs(w[1] - 4 / 3) < 1e-14
    x, w, _ = oracle.lgl(3)
    assert abs(x[1] + 1 / math.sqrt(5)) < 1e-14 and abs(w[0] - 1 / 6) < 1e-14
    assert abs(w[1] - 5 / 6) < 1e-14


@pytest.mark.parametrize("k", range(1, 21))
def test_lgl_invariants(k):
    x, w, D = oracle.lgl(k)
    assert x[0] == -1.0 and x[k] == 1.0 and np.all(np.diff(x) > 0) and np.all(w > 0)
    assert np.allclose(x, -x[::-1], atol=1e-15, rtol=0)
    assert abs(w.sum() - 2.0) < 2e-14
    assert np.abs(D @ np.ones(k + 1)).max() < 1e-12
    assert np.abs(D @ x - 1).max() < 1e-12


def test_lgl_invalid():
    with pytest.raises(ValueError):
        oracle.lgl(0)
    with pytest.raises(ValueError):
        oracle.lgl(21)


@pytest.mark.parametrize("k", [2, 5, 9, 16])
def test_diff_matrix_monomials(k):
    x, _, D = oracle.lgl(k)
    for j in range(k + 1):
        dxj = j * x ** (j - 1) if j else np.zeros_like(x)
        assert np.abs(D @ x ** j - dxj).max() < 1e-12


def test_gauss_quadrature():
    p, w = oracle.gauss(1)
    assert abs(p[0]) < 1e-15 and abs(w[0] - 2) < 1e-15
    p, w = oracle.gauss(2)
    assert abs(p[1] - 1 / math.sqrt(3)) < 1e-14 and abs(w[0] - 1) < 1e-14
    p, w = oracle.gauss(3)
    assert abs((w * p ** 4).sum() - 0.4) < 1e-14
    with pytest.raises(ValueError):
        oracle.gauss(0)


# ------------------------------------------------------------------ proj/tests/test_burgers.cpp
def test_burgers_flux_formulas():
    for a in (-1.3, 0.0, 0.7, 2.0):
        assert abs(oracle.burgers_flux("ef", a, a, 0, 0, 0.1) - a * a / 2) <= 1e-14 * max(1, a * a)
        assert abs(oracle.burgers_flux("lf", a, a, 0) - a * a / 2) <= 1e-14 * max(1, a * a)
    assert abs(oracle.burgers_flux("ef", 1, -1, 2, 0, 1) - 1 / 6) < 1e-15
    assert abs(oracle.burgers_flux("ef", 1, 0, 1, 3e-4, 0.05) - (1 / 6 + 0.006)) < 1e-13
    assert oracle.burgers_flux("lf", 2, 0, 2) == pytest.approx(3.0)


def test_burgers_gradient_exact_quadratic():
    # x(1-x) with zero Dirichlet data has the exact LDG gradient 1-2x
    P = oracle.Problem("burgers1d", 3, 5, box=(0, 1, 0, 1, 0, 1), periodic=False, kappa=0.1)
    x, _, _ = oracle.lgl(3)
    pts = np.concatenate([e / 5 + 0.5 * (x + 1) / 5 for e in range(5)])
    u = pts * (1 - pts)  # nodal interpolant equals the projection for a quadratic
    q, _ = oracle.burgers_diag(P, u, u)
    assert np.abs(q - (1 - 2 * pts)).max() < 1e-11


def test_burgers_linearity_and_invariance():
    rng = _rng(11)
    P = oracle.Problem("burgers1d", 4, 10, kappa=0.03)
    ref = rng.standard_normal(P.dim)
    for _ in range(5):
        u, w = rng.standard_normal(P.dim), rng.standard_normal(P.dim)
        lhs = P.apply_linear(ref, 1.7 * u - 0.4 * w)
        rhs = 1.7 * P.apply_linear(ref, u) - 0.4 * P.apply_linear(ref, w)
        assert np.linalg.norm(lhs - rhs) / (1 + np.linalg.norm(rhs)) < 1e-12
    for flux in ("lf", "ef"):
        for periodic in (True, False):
            P = oracle.Problem("burgers1d", 3, 9, kappa=0.02, flux=flux, sigma=1e-3, periodic=periodic)
            for _ in range(5):
                u = rng.standard_normal(P.dim)
                a, b = rng.standard_normal(P.dim), rng.standard_normal(P.dim)
                r1 = P.apply_linear(a, u) + P.apply_nonlinear(a, u)
                r2 = P.apply_linear(b, u) + P.apply_nonlinear(b, u)
                r3 = P.full_rhs(u)
                assert np.linalg.norm(r1 - r2) / np.linalg.norm(r1) < 1e-12
                assert np.linalg.norm(r1 - r3) / np.linalg.norm(r1) < 1e-12


def test_burgers_energy_identity_over_integrated():
    rng = _rng(42)
    for k in range(1, 7):
        P = oracle.Problem("burgers1d", k, 8, kappa=0.04, flux="ef", sigma=2e-3, over_integrate=True)
        for _ in range(5):
            u = rng.standard_normal(P.dim)
            _, (ip_ur, ip_qq, pen, ip_uu) = oracle.burgers_diag(P, u, u)
            assert abs(ip_ur + 0.04 * ip_qq + pen) <= 1e-10 * (1 + ip_uu)


# ------------------------------------------------------------------ proj/tests/test_euler.cpp
def _prim(rho, u, v, p, g=1.4):
    return np.array([rho, rho * u, rho * v, p / (g - 1) + 0.5 * rho * (u * u + v * v)])


def test_euler_flux_jacobian_fd_and_homogeneity():
    rng = _rng(17)
    for _ in range(20):
        q = _prim(rng.uniform(0.5, 2), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0.5, 2))
        a = rng.uniform(0, 2 * math.pi)
        n = (math.cos(a), math.sin(a))
        A = oracle.euler_pointwise(1, q, n=n).reshape(4, 4)
        F = lambda s: oracle.euler_pointwise(0, s)[:8].reshape(4, 2) @ np.array(n)
        for j in range(4):
            e = np.zeros(4); e[j] = 1e-6
            fd = (F(q + e) - F(q - e)) / 2e-6
            assert np.allclose(A[:, j], fd, rtol=1e-6, atol=1e-6)
        assert np.linalg.norm(A @ q - F(q)) / np.linalg.norm(F(q)) < 1e-12
    with pytest.raises(ArithmeticError):
        oracle.euler_pointwise(0, np.array([-1.0, 0, 0, 2.5]))


def test_euler_roe_and_lf_flux_properties():
    rng = _rng(37)
    for _ in range(10):
        qm = _prim(rng.uniform(0.5, 2), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0.5, 2))
        qp = _prim(rng.uniform(0.5, 2), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0.5, 2))
        a = rng.uniform(0, 2 * math.pi)
        n = (math.cos(a), math.sin(a))
        m = (-n[0], -n[1])
        for what in (2, 3):
            f1 = oracle.euler_pointwise(what, qm, qp, n)[:4]
            f2 = oracle.euler_pointwise(what, qp, qm, m)[:4]
            assert np.abs(f1 + f2).max() < 1e-12
            fe = oracle.euler_pointwise(what, qm, qm, n)[:4]
            ex = oracle.euler_pointwise(0, qm)[:8].reshape(4, 2) @ np.array(n)
            assert np.linalg.norm(fe - ex) / np.linalg.norm(ex) < 1e-13
    qm, qp = _prim(1, 0, 0, 1), _prim(4, 3, 0, 1)
    avg = oracle.euler_pointwise(5, qm, qp)
    assert abs(avg[0] - 2) < 1e-14 and abs(avg[1] - 2) < 1e-14


def test_euler_vortex_center_temperature():
    # default VortexParams (alpha 2, lambda 0.05, u_inf 0.2, xc 5, yc 0, wrap 10)
    q = oracle.vortex(5.0, 0.0, 0.0, [2.0, 0.05, 0.2, 0.0, 1, 1, 1, 5.0, 0.0, 10, 10])
    rho, u = q[0], q[1] / q[0]
    p = 0.4 * (q[3] - 0.5 * rho * u * u - 0.5 * q[2] ** 2 / rho)
    expect = 1.0 - (1.0 / 14.0) * (0.05 / (2 * math.pi)) ** 2 * math.exp(2.0)
    assert abs(p / rho - expect) < 1e-12 and abs(u - 0.2) < 1e-14


def test_euler_operator_uniform_flow_steady_and_invariance():
    for ef in ("roe", "lf"):
        P = oracle.Problem("euler2d", 2, 4, 4, box=(0, 10, -5, 5, 0, 1), euler_flux=ef)
        mean = _prim(1.0, 0.2, 0.0, 1.0)
        q = np.concatenate([np.repeat(mean[c], 9) for c in range(4)] * 16)
        assert np.abs(P.apply_linear(q, q) + P.apply_nonlinear(q, q)).max() < 1e-12
    rng = _rng(41)
    P = oracle.Problem("euler2d", 2, 3, 3, box=(0, 10, -5, 5, 0, 1), euler_flux="roe")

    def field():
        out = np.empty(P.dim)
        for e in range(9):
            for node in range(9):
                s = _prim(rng.uniform(0.5, 2), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0.5, 2))
                out[e * 36 + np.arange(4) * 9 + node] = s
        return out

    for _ in range(3):
        q = field()
        a, b = field(), field()
        r1 = P.apply_linear(a, q) + P.apply_nonlinear(a, q)
        r2 = P.apply_linear(b, q) + P.apply_nonlinear(b, q)
        assert np.linalg.norm(r1 - r2) / np.linalg.norm(r1) < 1e-11


# ------------------------------------------------------------------ proj/tests/test_phi.cpp
def matrix_with_spectrum(rng, n, lo, hi, nonnormality):
    t = np.diag(rng.uniform(lo, hi, n)) + np.triu(nonnormality * rng.standard_normal((n, n)), 1)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return q @ t @ q.T


def test_phi_scalar_special_values():
    for i in range(7):
        assert oracle.phi_scalar(i, 0.0) == pytest.approx(1 / math.factorial(i), rel=1e-15)
    assert oracle.phi_scalar(1, 1.0) == pytest.approx(math.e - 1, rel=1e-14)
    assert oracle.phi_scalar(2, 1.0) == pytest.approx(math.e - 2, rel=1e-13)


def test_expm_against_scipy():
    import scipy.linalg as sl
    rng = _rng(5)
    for scale in (1e-3, 0.1, 0.5, 1.5, 4.0, 60.0):
        A = rng.standard_normal((12, 12)) * scale / 3
        E = oracle.expm(A)
        R = sl.expm(A)
        assert np.abs(E - R).max() / np.abs(R).max() < 1e-12


def test_phi_combination_matches_dense_oracle():
    rng = _rng(2024)
    n = 50
    M = matrix_with_spectrum(rng, n, -20.0, 1.0, 1.0)
    b = [rng.standard_normal(n) for _ in range(4)]
    dt = 0.7
    fam = oracle.phi_dense_family(3, dt * M)
    expect = sum(dt ** i * fam[i] @ b[i] for i in range(4))
    got, iters, subs = oracle.phi_combination_dense(M, b, dt, tol=1e-10)
    assert np.linalg.norm(got - expect) / np.linalg.norm(expect) < 1e-8 and iters > 0


def test_krylov_build_relation_and_breakdown():
    rng = _rng(99)
    n = 30
    M = matrix_with_spectrum(rng, n, -5.0, 1.0, 1.0)
    V, H, m, inv, _ = oracle.krylov_build(M, rng.standard_normal(n), 20, 20)
    assert not inv and m == 20
    Vm = V[:, :20]
    assert np.abs(Vm.T @ Vm - np.eye(20)).max() < 1e-12
    assert np.abs(M @ Vm - V @ H).max() / np.linalg.norm(M) < 1e-10
    _, H1, m1, inv1, _ = oracle.krylov_build(np.eye(n), rng.standard_normal(n), 5, 5)
    assert m1 == 1 and inv1 and abs(H1[0, 0] - 1) < 1e-14
    with pytest.raises(ValueError):
        oracle.krylov_build(M, np.zeros(n), 3, 3)
