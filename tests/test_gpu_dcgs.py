"""GPU: the two orthogonalisations of fully orthogonalised phi calls (CGS2, DCGS2)
against the reference's two-pass modified Gram-Schmidt Arnoldi (proj/src/phi.cpp:84-112,
restated in the oracle) on the dense augmented operator [[dt L, dt r], [0, 0]] of a
stiff over-integrated Burgers problem (acceptance criterion 5's, Cr_d = 161), and
against each other on the full time loop."""
import math

import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import rel, to_dev, to_host

pytestmark = pytest.mark.gpu


def stiff_problem():
    u0, _, cfg = oracle.harness_burgers("burgers-smooth", 40, 4, "ef", 3e-4)
    kw = dict(box=(0.0, 1.0, 0, 1, 0, 1), periodic=False, kappa=cfg["kappa"], flux=cfg["flux"], sigma=cfg["sigma"],
              over_integrate=cfg["over_integrate"])
    return u0, pkg.OperatorSpec("burgers1d", 4, 40, **kw), oracle.Problem("burgers1d", 4, 40, **kw)


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2", "pdcgs2"])
@pytest.mark.parametrize("dt,m", [(1e-4, 16), (0.1, 40), (0.1, 80), (0.1, 128)])
def test_hessenberg_matches_mgs2(orth, dt, m):
    u0, spec, orc = stiff_problem()
    n = u0.size
    L = np.stack([orc.apply_linear(u0, np.eye(n)[i]) for i in range(n)], axis=1)
    r = orc.apply_linear(u0, u0) + orc.apply_nonlinear(u0, u0)
    aug = np.zeros((n + 1, n + 1))
    aug[:n, :n] = dt * L
    aug[:n, n] = dt * r
    seed = np.zeros(n + 1)
    seed[n] = 1.0
    _, href, _, _, _ = oracle.krylov_build(aug, seed, m, m)
    ctx = pkg.Context(0, orth="cgs2" if orth == "cgs2" else "dcgs2", pipelined=orth == "pdcgs2")
    op = pkg.Operator(ctx, spec)
    op.linearize(to_dev(u0))
    try:  # one substep: H is the first Arnoldi's (rejections halve h and reuse it)
        pkg.phi_combination(ctx, op, [None, to_dev(r)], dt, tol=1e-12, max_basis=m, orth_length=m, max_substeps=1)
    except pkg.KrylovError:
        pass
    h = ctx.debug_hessenberg()[:m + 1, :m]
    # the pipelined recurrence (one uninterrupted lookahead chain, grows included) on this stiff
    # operator (||dt A|| ~ 2.2e3): 7.9e-13 at m = 40, 3.2e-12 at 80, 1.6e-11 at 128 relative
    # (two-pass DCGS2 2.9e-12 at 128; tools/pipe_hess.py) -- C3-C5 stay at the DCGS2 level
    bar = 3e-11 if (orth == "pdcgs2" and m > 80) else 1e-11
    assert np.abs(h - href).max() <= bar * np.abs(href).max()


@pytest.mark.parametrize("pipelined", [False, True])
def test_dcgs2_and_cgs2_time_loops_agree(pipelined):
    u0, spec, _ = stiff_problem()
    out = {}
    for orth in ("cgs2", "dcgs2"):
        ctx = pkg.Context(0, orth=orth, pipelined=pipelined)
        op = pkg.Operator(ctx, spec)
        out[orth] = pkg.integrate(ctx, op, to_dev(u0), "epi2", 0.1, 1.0, tol=1e-12, max_basis=128, orth_length=128)
    a, b = out["cgs2"], out["dcgs2"]
    assert a.status == b.status == "completed"
    assert rel(to_host(b.u), to_host(a.u)) <= 1e-10
    assert list(a.iters_per_step) == list(b.iters_per_step)


@pytest.mark.parametrize("pipelined", [False, True])
def test_dcgs2_euler_matches_cgs2(pipelined):
    w = configs.scaled(configs.C4, 24, steps=3)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    res = {}
    for orth in ("cgs2", "dcgs2"):
        ctx = pkg.Context(0, orth=orth, pipelined=pipelined)
        res[orth] = pkg.integrate(ctx, pkg.Operator(ctx, w.spec()), to_dev(u0), "epi2", dt, w.steps * dt, tol=w.tol,
                                  max_basis=w.max_basis, orth_length=w.max_basis)
    assert rel(to_host(res["dcgs2"].u), to_host(res["cgs2"].u)) <= 1e-11
    assert list(res["dcgs2"].iters_per_step) == list(res["cgs2"].iters_per_step)


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2", "pdcgs2"])
def test_dense_fakes_with_breakdown(orth):
    # criterion-1 style dense fakes (proj/tests/acceptance.cpp:70-108) forced through each
    # orthogonalisation; n + p <= max_basis, so every call ends in a (lagged, for DCGS2)
    # happy breakdown at m = n + p
    from tests.gpu_util import matrix_with_spectrum
    rng = np.random.default_rng(77)
    ctx = pkg.Context(0, orth="cgs2" if orth == "cgs2" else "dcgs2", fused=False, pipelined=orth == "pdcgs2")
    worst = 0.0
    for trial in range(12):
        n = int(rng.integers(6, 60))
        M = matrix_with_spectrum(rng, n, -30.0, 2.0, 1.0)
        b = [rng.standard_normal(n) for _ in range(4)]
        fam = oracle.phi_dense_family(3, M)
        expect = sum(fam[i] @ b[i] for i in range(4))
        op = pkg.Operator(ctx, dense=M)
        got, st = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], 1.0, tol=1e-10)
        worst = max(worst, rel(to_host(got), expect))
        _, iters, subs = oracle.phi_combination_dense(M, b, 1.0, tol=1e-10)
        assert abs(st.iterations - iters) <= 1 and st.substeps == subs
    assert worst <= 1e-8
    # the identity: breakdown after one column
    op = pkg.Operator(ctx, dense=np.eye(8))
    b0 = rng.standard_normal(8)
    got, st = pkg.phi_combination(ctx, op, [to_dev(b0)], 0.5, tol=1e-12)
    assert rel(to_host(got), math.exp(0.5) * b0) < 1e-13


def _euler_run(monkeypatch, fused, max_basis, flux="lf"):
    # the strip JVP takes the DCGS2 pass-1 dots of columns j <= 43 in its own sweep
    # (EXPDG_E2_DOTS=0: the separate k_ts2 dots pass for every column); nx = 24 leaves a
    # partial last strip (10 + 10 + 4 elements)
    monkeypatch.setenv("EXPDG_E2_DOTS", fused)
    w = configs.scaled(configs.C4, 24, steps=3)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    spec = w.spec()
    if flux != "lf":
        spec = pkg.OperatorSpec("euler2d", spec.order, spec.nx, spec.ny, box=spec.box, euler_flux=flux)
    ctx = pkg.Context(0, orth="dcgs2", fused=False, pipelined=False)  # the two-pass DCGS2's fused sweep
    op = pkg.Operator(ctx, spec)
    res = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, w.steps * dt, tol=w.tol, max_basis=max_basis,
                        orth_length=max_basis)
    res.alg_bytes = ctx.traffic()["alg_bytes"]
    op.linearize(to_dev(u0))
    r = to_dev(to_host(op.apply_linear(to_dev(u0))) + to_host(op.apply_nonlinear(to_dev(u0))))
    try:  # one substep at 2x dt: H of one Arnoldi with columns past the fused bound
        pkg.phi_combination(ctx, op, [None, r], 2 * dt, tol=1e-14, max_basis=max_basis, orth_length=max_basis,
                            max_substeps=1)
    except pkg.KrylovError:
        pass
    return res, ctx.debug_hessenberg()[:max_basis + 1, :max_basis]


@pytest.mark.parametrize("max_basis,flux", [(40, "lf"), (64, "lf"), (40, "roe")])
def test_euler_fused_dots_match_dots_pass(monkeypatch, max_basis, flux):
    a, ha = _euler_run(monkeypatch, "1", max_basis, flux)
    b, hb = _euler_run(monkeypatch, "0", max_basis, flux)
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)
    assert np.abs(ha - hb).max() <= 1e-12 * np.abs(hb).max()
    # the sweep really took the dots: u and w are not re-read (16 n bytes less per column)
    assert a.alg_bytes < b.alg_bytes


@pytest.mark.parametrize("orth", ["dcgs2", "cgs2", "pdcgs2"])
def test_host_stepped_cycles_match_graph(orth):
    # host-stepped loops launch only the kernels that do work in a cycle (the host reads back
    # the next action and column); the graph launches every kernel and lets them no-op.  Both
    # must give the same bits; max_basis 64 crosses the fused-dots bound (columns j > 33)
    w = configs.scaled(configs.C4, 24, steps=2)
    u0 = w.initial_condition()
    dt = 2 * w.time_step(u0)
    out = []
    for graph in (True, False):
        ctx = pkg.Context(0, orth="cgs2" if orth == "cgs2" else "dcgs2", fused=False, pipelined=orth == "pdcgs2")
        op = pkg.Operator(ctx, w.spec())
        out.append(pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, w.steps * dt, tol=1e-12, max_basis=64,
                                 orth_length=64, use_graph=graph))
    a, b = out
    assert a.status == b.status == "completed"
    assert np.array_equal(to_host(a.u), to_host(b.u))
    assert list(a.iters_per_step) == list(b.iters_per_step)
    assert max(np.diff(np.concatenate([[0], a.iters_per_step]))) > 34  # columns past the fused bound


@pytest.mark.parametrize("n,max_basis", [(4, 40), (6, 64)])
def test_euler3d_fused_dots_match_dots_pass(monkeypatch, n, max_basis):
    # the 3D z-march takes the DCGS2 pass-1 dots of columns j <= 43 in its own sweep on meshes
    # of whole 2x2 tiles (EXPDG_E3_DOTS=0: the separate k_ts2 dots pass)
    w = configs.scaled(configs.C5, n, steps=2)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    out = []
    for v in ("1", "0"):
        monkeypatch.setenv("EXPDG_E3_DOTS", v)
        ctx = pkg.Context(0, orth="dcgs2", fused=False, pipelined=False)
        op = pkg.Operator(ctx, w.spec())
        r = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, w.steps * dt, tol=w.tol, max_basis=max_basis,
                          orth_length=max_basis)
        r.alg_bytes = ctx.traffic()["alg_bytes"]
        out.append(r)
    a, b = out
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)
    assert a.alg_bytes < b.alg_bytes  # the sweep took the dots


@pytest.mark.parametrize("kind,nx", [("C4", 24), ("C3", 32), ("C5", 6)])
def test_pipelined_dcgs2_matches_two_pass(kind, nx):
    # pipelined DCGS2 (one basis stream per column: the lookahead application + k_ts3) against the
    # two-pass DCGS2 on the same trajectory: same Krylov dimensions, solutions to rounding, and the
    # algorithm moves fewer bytes (8 n (j + 10) instead of 8 n (2 j + 8) per column)
    w = configs.scaled(configs.ALL[kind], nx, steps=3)
    u0 = w.initial_condition()
    dt = w.time_step(u0) if w.dt is None else w.dt
    out = []
    for pipe in (True, False):
        ctx = pkg.Context(0, orth="dcgs2", pipelined=pipe)
        r = pkg.integrate(ctx, pkg.Operator(ctx, w.spec()), to_dev(u0), "epi2", dt, w.steps * dt, tol=w.tol,
                          max_basis=w.max_basis, orth_length=w.max_basis)
        r.alg_bytes = ctx.traffic()["alg_bytes"]
        r.path = ctx.last_path()
        out.append(r)
    a, b = out
    assert a.path["pipelined"] and not b.path["pipelined"]
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)
    assert a.alg_bytes < b.alg_bytes
