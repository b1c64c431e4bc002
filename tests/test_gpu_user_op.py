"""GPU parity of the completed drop-in boundary (include/expdg_b200.h):

* a user LinearAction / SplitProblem (proj/include/expdg/phi.hpp:11,
  proj/include/expdg/integrators.hpp:48-52) — neither dense nor one of the built-in DG
  operators: a matrix-free finite-difference viscous Burgers split written with torch ops —
  drives the device phi engine (`phi_combination`) and time loop (`integrate`), host-stepped
  and graph-recorded (graph_safe), against the oracle running the same split through the
  reference algorithm (oracle.phi_combination_user / oracle.integrate_user);
* `krylov_build` (proj/src/phi.cpp:115-130) on the device vs the oracle;
* TimeLoopConfig::snapshot_every / on_step (proj/include/expdg/integrators.hpp:58-63,
  proj/src/integrators.cpp:186-197) vs the oracle.
"""
import math

import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import matrix_with_spectrum, oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu

N = 256
NU = 0.02
H = 2 * math.pi / N


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def fd_numpy():
    """Periodic central-difference viscous Burgers f(u) = -(u^2/2)_x + nu u_xx, split at ref:
    L = f'(ref), N = f - L (the reference's splitting convention, proj/src/burgers.cpp:309-320)."""
    def d1(v):
        return (np.roll(v, -1) - np.roll(v, 1)) / (2 * H)

    def d2(v):
        return (np.roll(v, -1) - 2.0 * v + np.roll(v, 1)) / (H * H)

    def linearize(ref):
        if not np.all(np.isfinite(ref)):
            raise ValueError("non-finite reference")
        if np.max(np.abs(ref)) > 50.0:
            raise ArithmeticError("inadmissible reference")
        r = ref.copy()
        lin = lambda x: -d1(r * x) + NU * d2(x)  # noqa: E731
        non = lambda x: -d1(0.5 * x * x) + NU * d2(x) - lin(x)  # noqa: E731
        return lin, non
    return linearize


def fd_torch():
    import torch

    def d1(v):
        return (torch.roll(v, -1) - torch.roll(v, 1)) / (2 * H)

    def d2(v):
        return (torch.roll(v, -1) - 2.0 * v + torch.roll(v, 1)) / (H * H)

    def linearize(ref):
        if not bool(torch.isfinite(ref).all()):
            raise ValueError("non-finite reference")
        if float(ref.abs().max()) > 50.0:
            raise ArithmeticError("inadmissible reference")
        r = ref.clone()
        lin = lambda x: -d1(r * x) + NU * d2(x)  # noqa: E731
        non = lambda x: -d1(0.5 * x * x) + NU * d2(x) - lin(x)  # noqa: E731
        return lin, non
    return linearize


def fd_torch_graph_safe():
    """The same split as allocation-free (x, out) actions on preallocated buffers, so the
    library may record them once into its CUDA graphs (graph_safe)."""
    import torch
    dev = "cuda:0"
    ref = torch.zeros(N, dtype=torch.float64, device=dev)
    a = torch.zeros(N, dtype=torch.float64, device=dev)
    b = torch.zeros(N, dtype=torch.float64, device=dev)

    def flux_form(v, out, nu_part_of):
        # out = -d1(v) + nu d2(nu_part_of), periodic, in place on slices
        torch.sub(v[2:], v[:-2], out=out[1:-1])
        torch.sub(v[1:2], v[-1:], out=out[:1])
        torch.sub(v[:1], v[-2:-1], out=out[-1:])
        out.mul_(-1.0 / (2 * H))
        x = nu_part_of
        torch.add(x[2:], x[:-2], out=b[1:-1])
        torch.add(x[1:2], x[-1:], out=b[:1])
        torch.add(x[:1], x[-2:-1], out=b[-1:])
        b.sub_(x, alpha=2.0)
        out.add_(b, alpha=NU / (H * H))

    def lin(x, out):
        torch.mul(ref, x, out=a)
        flux_form(a, out, x)

    def non(x, out):
        # f(x) - L x = -d1(x^2/2 - ref x)
        torch.mul(x, x, out=a)
        a.mul_(0.5)
        a.addcmul_(ref, x, value=-1.0)
        torch.sub(a[2:], a[:-2], out=out[1:-1])
        torch.sub(a[1:2], a[-1:], out=out[:1])
        torch.sub(a[:1], a[-2:-1], out=out[-1:])
        out.mul_(-1.0 / (2 * H))

    def linearize(r):
        ref.copy_(r)
        return lin, non
    return linearize


def u0_profile():
    x = np.arange(N) * H
    return 0.5 + np.sin(x) + 0.2 * np.cos(3 * x)


def _dims(r):
    return np.diff(np.concatenate([[0], np.asarray(r.iters_per_step)]))


@pytest.mark.parametrize("graph_safe", [False, True])
def test_user_linear_action_phi_matches_oracle(ctx, graph_safe):
    rng = np.random.default_rng(11)
    ref = u0_profile()
    L_np, _ = fd_numpy()(ref)
    lz = fd_torch_graph_safe() if graph_safe else fd_torch()
    prob = pkg.SplitProblem(N, linearize=lz, graph_safe=graph_safe)
    op = pkg.UserOperator(ctx, prob)
    op.linearize(to_dev(ref))
    b = [rng.standard_normal(N) for _ in range(3)]
    dt = 0.05
    got, st = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], dt, tol=1e-10, max_basis=40, orth_length=40)
    exp_, iters, subs = oracle.phi_combination_user(L_np, N, b, dt, tol=1e-10, max_basis=40, orth_length=40)
    assert rel(to_host(got), exp_) <= 1e-10
    assert abs(st.iterations - iters) <= 1 and st.substeps == subs
    assert ctx.last_path()["graph"] is graph_safe


def test_user_op_apply_matches_numpy(ctx):
    rng = np.random.default_rng(5)
    ref = u0_profile()
    x = rng.standard_normal(N)
    L_np, N_np = fd_numpy()(ref)
    op = pkg.UserOperator(ctx, pkg.SplitProblem(N, linearize=fd_torch()))
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), L_np(x)) < 1e-14
    assert rel(to_host(op.apply_nonlinear(to_dev(x))), N_np(x)) < 1e-14


@pytest.mark.parametrize("graph_safe", [False, True])
@pytest.mark.parametrize("integ", ["epi2", "exprb42", "exp_euler"])
def test_user_split_problem_integrate_matches_oracle(ctx, integ, graph_safe):
    u0 = u0_profile()
    dt, steps = 0.02, 6
    kw = dict(tol=1e-10, max_basis=30, orth_length=30)
    orc = oracle.integrate_user(N, fd_numpy(), integ, u0, dt, steps * dt, snapshot_every=2, **kw)
    lz = fd_torch_graph_safe() if graph_safe else fd_torch()
    op = pkg.UserOperator(ctx, pkg.SplitProblem(N, linearize=lz, graph_safe=graph_safe))
    seen = []
    r = pkg.integrate(ctx, op, to_dev(u0), integ, dt, steps * dt, snapshot_every=2,
                      on_step=lambda *a: seen.append(a), **kw)
    assert r.status == orc.status == "completed" and r.steps == orc.steps == steps
    assert rel(to_host(r.u), orc.u) <= 1e-9
    assert np.max(np.abs(_dims(r) - _dims(orc))) <= 1
    assert len(r.snapshots) == len(orc.snapshots) == 3
    for (t_d, u_d), (t_o, u_o) in zip(r.snapshots, orc.snapshots):
        assert t_d == t_o
        assert rel(to_host(u_d), u_o) <= 1e-9
    assert [s[0] for s in seen] == list(range(1, steps + 1))
    assert np.allclose([s[1] for s in seen], np.cumsum([dt] * steps), rtol=0, atol=1e-15)
    assert [s[3] for s in seen] == list(r.iters_per_step)
    assert ctx.last_path()["graph"] is graph_safe


def test_user_split_domain_error_blows_up_like_reference(ctx):
    # linearize raising domain_error inside the loop -> blew_up at that step (proj/src/integrators.cpp:179-193)
    u0 = u0_profile()
    u0[7] = 60.0  # the split's admissibility bound is 50
    kw = dict(tol=1e-10, max_basis=30, orth_length=30)
    orc = oracle.integrate_user(N, fd_numpy(), "epi2", u0, 0.01, 0.05, **kw)
    op = pkg.UserOperator(ctx, pkg.SplitProblem(N, linearize=fd_torch()))
    seen = []
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", 0.01, 0.05, on_step=lambda *a: seen.append(a), **kw)
    assert orc.status == r.status == "blew_up" and r.blow_up_step == orc.blow_up_step == 1
    assert seen == []
    # invalid_argument propagates out of integrate, as in the reference
    u1 = u0_profile()
    u1[3] = np.nan
    with pytest.raises(ValueError):
        pkg.integrate(ctx, op, to_dev(u1), "epi2", 0.01, 0.05, **kw)


@pytest.mark.parametrize("m,orth", [(1, 10), (12, 12), (30, 30), (20, 5)])
def test_krylov_build_matches_oracle(ctx, m, orth):
    # proj/tests/test_phi.cpp:124-163 style: dense fake and the user operator
    rng = np.random.default_rng(100 + m)
    n = 60
    A = matrix_with_spectrum(rng, n, -10.0, 1.0, 0.5)
    seed = rng.standard_normal(n)
    V, Hm, k, inv, sn = oracle.krylov_build(A, seed, m, orth)
    f = pkg.krylov_build(ctx, pkg.Operator(ctx, dense=A), to_dev(seed), m, orth)
    assert f.m == k and f.invariant_subspace == inv
    assert abs(f.seed_norm - sn) <= 1e-14 * sn
    assert rel(f.hessenberg, Hm) <= 1e-11
    assert rel(to_host(f.basis), V) <= 1e-11
    # the Arnoldi relation on the device basis: A V_m = V_{m+1} H
    Vd = to_host(f.basis)
    assert rel(A @ Vd[:, :k], Vd @ f.hessenberg) <= 1e-11


def test_krylov_build_invariant_subspace_and_zero_seed(ctx):
    # identity: breakdown after one column (proj/tests/test_phi.cpp:139-146); zero seed throws (:162)
    n = 20
    rng = np.random.default_rng(3)
    f = pkg.krylov_build(ctx, pkg.Operator(ctx, dense=np.eye(n)), to_dev(rng.standard_normal(n)), 5, 5)
    assert f.m == 1 and f.invariant_subspace and f.basis.shape == (n, 1)
    with pytest.raises(ValueError):
        pkg.krylov_build(ctx, pkg.Operator(ctx, dense=np.eye(n)), to_dev(np.zeros(n)), 3, 3)


def test_krylov_build_on_user_operator_matches_oracle(ctx):
    ref = u0_profile()
    L_np, _ = fd_numpy()(ref)
    A = np.stack([L_np(e) for e in np.eye(N)], axis=1)
    # a generic seed: a smooth one leaves the late Krylov directions at rounding level (ill-determined H)
    seed = np.random.default_rng(8).standard_normal(N)
    V, Hm, k, inv, sn = oracle.krylov_build(A, seed, 25, 25)
    op = pkg.UserOperator(ctx, pkg.SplitProblem(N, linearize=fd_torch()))
    op.linearize(to_dev(ref))
    f = pkg.krylov_build(ctx, op, to_dev(seed), 25, 25)
    assert f.m == k == 25
    assert rel(f.hessenberg, Hm) <= 1e-10


def test_snapshots_and_on_step_builtin_operator(ctx):
    # C4 physics on a reduced mesh, graph control: snapshots every 2 steps vs the oracle's
    w = configs.scaled(configs.C4, 8, steps=5)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    orc = oracle_problem(w.spec()).integrate("epi2", u0, dt, 5 * dt, snapshot_every=2, **kw)
    op = pkg.Operator(ctx, w.spec())
    seen = []
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, 5 * dt, snapshot_every=2, on_step=lambda *a: seen.append(a),
                      **kw)
    assert len(r.snapshots) == len(orc.snapshots) == 2
    for (t_d, u_d), (t_o, u_o) in zip(r.snapshots, orc.snapshots):
        assert t_d == t_o and rel(to_host(u_d), u_o) <= 1e-9
    assert [s[0] for s in seen] == [1, 2, 3, 4, 5]
    assert np.allclose([s[2] for s in seen], orc.amax_per_step, rtol=1e-9)
    # host buffers: same snapshots through expdg_integrate_host
    rh = pkg.integrate(ctx, op, u0.copy(), "epi2", dt, 5 * dt, snapshot_every=2, **kw)
    for (t_d, u_d), (t_h, u_h) in zip(r.snapshots, rh.snapshots):
        assert t_d == t_h and np.array_equal(to_host(u_d), u_h)
