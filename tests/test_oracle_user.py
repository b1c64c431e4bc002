"""The oracle's user-callback entry points (oracle_phi_user / oracle_integrate_user, the
checker of the device user-operator path) run the same reference algorithm as its built-in
problems: a SplitProblem whose linearize returns the built-in operator's own L / N must
reproduce the built-in integrate bit for bit, snapshots included (proj/src/integrators.cpp:195-196)."""
import numpy as np

import oracle
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem


def test_integrate_user_reproduces_builtin_problem():
    w = configs.scaled(configs.C1_S3E4, 16, steps=4)
    u0 = oracle.initial_condition(w.config, w.nx, w.order, configs.SEEDS[w.config], w.noise)
    P = oracle_problem(w.spec())
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    ref = P.integrate("epi2", u0, w.dt, 4 * w.dt, snapshot_every=2, **kw)

    def linearize(r):
        r = r.copy()
        return (lambda x: P.apply_linear(r, x)), (lambda x: P.apply_nonlinear(r, x))

    got = oracle.integrate_user(P.dim, linearize, "epi2", u0, w.dt, 4 * w.dt, snapshot_every=2, **kw)
    assert got.status == ref.status == "completed"
    assert np.array_equal(got.u, ref.u)
    assert np.array_equal(got.iters_per_step, ref.iters_per_step)
    assert len(got.snapshots) == len(ref.snapshots) == 2
    for (ta, ua), (tb, ub) in zip(got.snapshots, ref.snapshots):
        assert ta == tb and np.array_equal(ua, ub)
    assert np.array_equal(ref.snapshots[-1][1], ref.u)


def test_phi_user_matches_dense():
    rng = np.random.default_rng(4)
    A = -np.diag(rng.uniform(0, 20, 30)) + 0.1 * rng.standard_normal((30, 30))
    b = [rng.standard_normal(30) for _ in range(3)]
    a = oracle.phi_combination_user(lambda x: A @ x, 30, b, 0.3, tol=1e-10)
    d = oracle.phi_combination_dense(A, b, 0.3, tol=1e-10)
    assert a[1:] == d[1:]
    assert np.allclose(a[0], d[0], rtol=1e-13, atol=1e-13)


def test_integrate_user_domain_error_is_blow_up():
    def linearize(r):
        if r[0] > 1.0:
            raise ArithmeticError("inadmissible")
        return (lambda x: -x), None

    u0 = np.full(8, 2.0)
    r = oracle.integrate_user(8, linearize, "epi2", u0, 0.1, 0.3, tol=1e-10, max_basis=8, orth_length=8)
    assert r.status == "blew_up" and r.blow_up_step == 1
