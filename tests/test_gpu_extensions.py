"""GPU parity for the configs outside the reference's dimensionality:
C3 (2D tensor-product LDG Burgers) and C5 (3D Lax-Friedrichs Euler).  Each is
checked against its oracle definition, reduces to the reference-matched lower-
dimensional device operator, and (C5) converges at design order on the exact
isentropic vortex."""
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


# ------------------------------------------------------------------ 2D Burgers
@pytest.mark.parametrize("order,nx,ny,periodic,flux,sigma", [
    (4, 6, 5, True, "lf", 0.0),
    (3, 4, 7, False, "ef", 1e-3),
    (2, 5, 5, True, "ef", 0.5),
    (7, 3, 2, True, "lf", 0.0),
])
def test_burgers2d_apply_matches_oracle(ctx, order, nx, ny, periodic, flux, sigma):
    rng = np.random.default_rng(order + 10 * nx)
    spec = pkg.OperatorSpec("burgers2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), periodic=periodic, kappa=1e-2,
                            flux=flux, sigma=sigma)
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    ref, x = rng.standard_normal(op.dim), rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < 1e-13
    assert rel(to_host(op.apply_nonlinear(to_dev(x))), orc.apply_nonlinear(ref, x)) < 1e-13
    assert rel(to_host(op.full_rhs(to_dev(x))), orc.full_rhs(x)) < 1e-13


def test_burgers2d_y_invariant_reduces_to_1d(ctx):
    # a y-invariant field: the 2D operator equals the reference-matched 1D operator on every line
    order, nx, ny = 4, 16, 3
    rng = np.random.default_rng(3)
    s1 = pkg.OperatorSpec("burgers1d", order, nx, box=(0, 2 * math.pi, 0, 1, 0, 1), kappa=1e-2, flux="ef", sigma=0.3)
    s2 = pkg.OperatorSpec("burgers2d", order, nx, ny, box=(0, 2 * math.pi, 0, 1, 0, 1), kappa=1e-2, flux="ef",
                          sigma=0.3)
    op1, op2 = pkg.Operator(ctx, s1), pkg.Operator(ctx, s2)
    np1 = order + 1
    u1, x1 = rng.standard_normal(op1.dim), rng.standard_normal(op1.dim)

    def extrude(v):
        out = np.empty(op2.dim)
        blk = out.reshape(ny, nx, np1, np1)  # [je][ie][j][i]
        blk[:] = v.reshape(nx, np1)[None, :, None, :]
        return out

    op1.linearize(to_dev(u1))
    op2.linearize(to_dev(extrude(u1)))
    for f1, f2 in ((op1.apply_linear, op2.apply_linear), (op1.apply_nonlinear, op2.apply_nonlinear),
                   (op1.full_rhs, op2.full_rhs)):
        y1 = to_host(f1(to_dev(x1)))
        y2 = to_host(f2(to_dev(extrude(x1))))
        assert np.abs(y2 - extrude(y1)).max() <= 1e-12 * np.abs(y1).max()


def test_c3_reduced_mesh_epi2_parity(ctx):
    w = configs.scaled(configs.C3, 16, steps=3)
    u0 = w.initial_condition()
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, w.steps * w.dt, tol=w.tol, max_basis=w.max_basis,
                                             orth_length=w.max_basis)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", w.dt, w.steps * w.dt, tol=w.tol, max_basis=w.max_basis,
                      orth_length=w.max_basis)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1


# ------------------------------------------------------------------ 3D Euler
def random_state5(rng, ne, npe):
    q = np.empty(ne * 5 * npe)
    for e in range(ne):
        rho = rng.uniform(0.5, 2.0, npe)
        vel = [rng.uniform(-1, 1, npe) for _ in range(3)]
        p = rng.uniform(0.5, 2.0, npe)
        blk = q[e * 5 * npe:(e + 1) * 5 * npe].reshape(5, npe)
        blk[0] = rho
        for d in range(3):
            blk[1 + d] = rho * vel[d]
        blk[4] = p / 0.4 + 0.5 * rho * sum(v * v for v in vel)
    return q


@pytest.mark.parametrize("order,n", [(1, 3), (2, 3), (3, 2), (4, 2), (5, 2)])
def test_euler3d_apply_matches_oracle(ctx, order, n):
    rng = np.random.default_rng(order)
    spec = pkg.OperatorSpec("euler3d", order, n, n + 1, n, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    op = pkg.Operator(ctx, spec)
    orc = oracle_problem(spec)
    npe = (order + 1) ** 3
    ne = n * (n + 1) * n
    ref, q = random_state5(rng, ne, npe), random_state5(rng, ne, npe)
    x = rng.standard_normal(op.dim)
    op.linearize(to_dev(ref))
    assert rel(to_host(op.apply_linear(to_dev(x))), orc.apply_linear(ref, x)) < 1e-13
    assert rel(to_host(op.apply_nonlinear(to_dev(q))), orc.apply_nonlinear(ref, q)) < 1e-13
    assert rel(to_host(op.full_rhs(to_dev(q))), orc.full_rhs(q)) < 1e-12


def test_euler3d_z_invariant_reduces_to_2d(ctx):
    order, nx, ny, nz = 3, 4, 3, 2
    rng = np.random.default_rng(5)
    s2 = pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 10, 0, 6, 0, 1), euler_flux="lf")
    s3 = pkg.OperatorSpec("euler3d", order, nx, ny, nz, box=(0, 10, 0, 6, 0, 2), euler_flux="lf")
    op2, op3 = pkg.Operator(ctx, s2), pkg.Operator(ctx, s3)
    np1 = order + 1
    n2 = np1 * np1

    def state2(rng):
        q = np.empty(nx * ny * 4 * n2)
        for e in range(nx * ny):
            rho, u, v, p = (rng.uniform(0.5, 2, n2), rng.uniform(-1, 1, n2), rng.uniform(-1, 1, n2),
                            rng.uniform(0.5, 2, n2))
            blk = q[e * 4 * n2:(e + 1) * 4 * n2].reshape(4, n2)
            blk[0], blk[1], blk[2], blk[3] = rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)
        return q

    def extrude(q2, zero_w=True):
        out = np.zeros(op3.dim)
        b3 = out.reshape(nz, ny, nx, 5, np1, np1, np1)  # [kz][jy][ix][c][k][j][i]
        b2 = q2.reshape(ny, nx, 4, np1, np1)
        for c2, c3 in ((0, 0), (1, 1), (2, 2), (3, 4)):
            b3[:, :, :, c3] = b2[None, :, :, c2, None, :, :]
        return out

    def project(y3):  # 3D result restricted to the 2D components of the kz=0, k=0 plane
        b3 = y3.reshape(nz, ny, nx, 5, np1, np1, np1)
        out = np.empty((ny, nx, 4, np1, np1))
        for c2, c3 in ((0, 0), (1, 1), (2, 2), (3, 4)):
            out[:, :, c2] = b3[0, :, :, c3, 0]
        return out.reshape(-1), b3[:, :, :, 3]

    ref, x, q = state2(rng), rng.standard_normal(op2.dim), state2(rng)
    op2.linearize(to_dev(ref))
    op3.linearize(to_dev(extrude(ref)))
    for name in ("apply_linear", "apply_nonlinear", "full_rhs"):
        arg2 = x if name == "apply_linear" else q
        y2 = to_host(getattr(op2, name)(to_dev(arg2)))
        y3 = to_host(getattr(op3, name)(to_dev(extrude(arg2))))
        proj, wmom = project(y3)
        scale = np.abs(y2).max()
        assert np.abs(proj - y2).max() <= 1e-12 * scale, name
        assert np.abs(wmom).max() <= 1e-12 * scale, name


def test_c5_reduced_mesh_epi2_parity(ctx):
    w = configs.scaled(configs.C5, 4, steps=2)
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


@pytest.mark.parametrize("order", [4, 5])
def test_euler3d_orders_4_5_epi2_parity(ctx, order):
    # orders above C5's run the element-tile kernels (125 / 216 nodes per element: 2 / 1 elements
    # per CTA); EPI2 against the oracle on a 2 x 3 x 2 mesh
    rng = np.random.default_rng(order)
    spec = pkg.OperatorSpec("euler3d", order, 2, 3, 2, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    op = pkg.Operator(ctx, spec)
    u0 = random_state5(rng, 12, (order + 1) ** 3)
    kw = dict(tol=1e-10, max_basis=20, orth_length=20)
    r = pkg.integrate(ctx, op, to_dev(u0), "epi2", 1e-4, 3e-4, **kw)
    orc = oracle_problem(spec).integrate("epi2", u0, 1e-4, 3e-4, **kw)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1


def _vortex(x, y, t, lam=0.05, alpha=2.0, uinf=0.2, xc=5.0, yc=0.0, gamma=1.4):
    # proj/src/euler.cpp:160-184 with the reference default VortexParams
    cp = gamma / (gamma - 1.0)
    xt = x - xc - uinf * t
    yt = y - yc
    xt = xt - 10.0 * np.round(xt / 10.0)
    yt = yt - 10.0 * np.round(yt / 10.0)
    r2 = xt * xt + yt * yt
    s = lam / (2 * math.pi)
    e1 = np.exp(0.5 * alpha * (1 - r2))
    u = uinf - s * yt * e1
    v = s * xt * e1
    T = 1.0 - s * s / (2 * alpha * cp) * np.exp(alpha * (1 - r2))
    rho = T ** (1 / (gamma - 1))
    p = T ** (gamma / (gamma - 1))
    return rho, u, v, p


def test_c5_extruded_vortex_converges_at_design_order(ctx):
    # 3D operator on a z-extruded exact isentropic vortex: L2 error at t = 0.5 decays at
    # (about) the design order k+1 under h-refinement (k = 3, dt small).
    order = 3
    np1 = order + 1
    x_lgl, w_lgl, _ = pkg.lgl_basis(order)
    errs = []
    hs = []
    for n in (4, 8):
        nz = 1
        spec = pkg.OperatorSpec("euler3d", order, n, n, nz, box=(0, 10, -5, 5, 0, 1), euler_flux="lf")
        op = pkg.Operator(ctx, spec)
        h = 10.0 / n
        xe = (np.arange(n)[:, None] + 0.5 * (x_lgl[None, :] + 1)) * h        # [ie][i]
        ye = -5 + (np.arange(n)[:, None] + 0.5 * (x_lgl[None, :] + 1)) * h   # [je][j]
        X = xe[None, :, None, :]  # [je][ie][j][i]
        Y = ye[:, None, :, None]

        def state(t):
            rho, u, v, p = _vortex(np.broadcast_to(X, (n, n, np1, np1)), np.broadcast_to(Y, (n, n, np1, np1)), t)
            q = np.zeros((nz, n, n, 5, np1, np1, np1))
            comps = [rho, rho * u, rho * v, 0 * rho, p / 0.4 + 0.5 * rho * (u * u + v * v)]
            for c in range(5):
                q[:, :, :, c] = comps[c].transpose(0, 1, 2, 3)[None, :, :, None, :, :]
            return q.reshape(-1)

        t_end, dt = 0.5, 0.05
        r = pkg.integrate(ctx, op, to_dev(state(0.0)), "epi2", dt, t_end, tol=1e-12, max_basis=40, orth_length=40)
        assert r.status == "completed"
        d = (to_host(r.u) - state(t_end)).reshape(nz, n, n, 5, np1, np1, np1)[:, :, :, 0]
        wq = (w_lgl[:, None, None] * w_lgl[None, :, None] * w_lgl[None, None, :]) * (h * h * 1.0) / 8.0
        errs.append(math.sqrt(float(np.sum(d * d * wq[None, None, None]))))
        hs.append(h)
    order_obs = math.log(errs[0] / errs[1]) / math.log(hs[0] / hs[1])
    assert order_obs >= order + 0.5, (errs, order_obs)


def _plane_vortex_errors(ctx, plane, sizes, order=3, t_end=0.5, dt=0.05):
    """Density L2 errors of the exact vortex laid in the given coordinate plane (the third axis one
    element wide, the solution constant along it) after EPI2 to t_end, one per mesh size."""
    np1 = order + 1
    x_lgl, w_lgl, _ = pkg.lgl_basis(order)
    ax = {"x": 2, "y": 1, "z": 0}  # element axis of [kz][jy][ix], node axis = 4 + the same
    errs = []
    for n in sizes:
        h = 10.0 / n
        a = (np.arange(n)[:, None] + 0.5 * (x_lgl[None, :] + 1)) * h        # first in-plane coordinate [e][node]
        b = -5 + (np.arange(n)[:, None] + 0.5 * (x_lgl[None, :] + 1)) * h   # second
        dims = {c: (n if c in plane else 1) for c in "xyz"}
        box = []
        for c in "xyz":
            box += ([0, 10] if c == plane[0] else [-5, 5]) if c in plane else [0, 1]
        spec = pkg.OperatorSpec("euler3d", order, dims["x"], dims["y"], dims["z"], box=tuple(box), euler_flux="lf")
        shape = (dims["z"], dims["y"], dims["x"], 5, np1, np1, np1)  # [kz][jy][ix][c][k][j][i]
        full = shape[:3] + shape[4:]

        def coord(vals, c):
            idx = [None] * 6
            idx[ax[c]] = slice(None)
            idx[3 + ax[c]] = slice(None)
            return np.broadcast_to(vals[tuple(idx)], full)

        A, B = coord(a, plane[0]), coord(b, plane[1])
        op = pkg.Operator(ctx, spec)

        def state(t):
            rho, u1, u2, p = _vortex(A, B, t)
            q = np.zeros(shape)
            mom = {c: 0 * rho for c in "xyz"}
            mom[plane[0]], mom[plane[1]] = rho * u1, rho * u2
            comps = [rho, mom["x"], mom["y"], mom["z"], p / 0.4 + 0.5 * rho * (u1 * u1 + u2 * u2)]
            for c in range(5):
                q[:, :, :, c] = comps[c]
            return q.reshape(-1)

        r = pkg.integrate(ctx, op, to_dev(state(0.0)), "epi2", dt, t_end, tol=1e-12, max_basis=40, orth_length=40)
        assert r.status == "completed"
        d = (to_host(r.u) - state(t_end)).reshape(shape)[:, :, :, 0]
        wq = (w_lgl[:, None, None] * w_lgl[None, :, None] * w_lgl[None, None, :]) * (h * h * 1.0) / 8.0
        errs.append(math.sqrt(float(np.sum(d * d * wq[None, None, None]))))
    return errs


@pytest.mark.parametrize("plane", ["xz", "yz"])
def test_c5_vortex_in_a_z_plane_converges_like_the_xy_plane(ctx, plane):
    # The exact vortex laid in the x-z (y-z) plane, so the z-derivatives, the z-faces and the
    # w-momentum carry the solution and the z direction is refined: the design-order check of the
    # test above (k = 3, meshes 4 and 8 as the reference's criterion 8 takes h and h / 2; observed
    # 4.8 here) must hold there too, and the errors must equal those of the x-y plane (the 3D
    # operator treats the three directions alike; measured equal to every printed digit).
    ref = _plane_vortex_errors(ctx, "xy", (4, 8))
    errs = _plane_vortex_errors(ctx, plane, (4, 8))
    order_obs = math.log(errs[0] / errs[1]) / math.log(2.0)
    assert order_obs >= 3.5, (errs, order_obs)
    for e, r in zip(errs, ref):
        assert abs(e - r) <= 1e-9 * r, (errs, ref)


# ------------------------------------------------------------------ strip / z-march phi kernels
def _two_kernels(monkeypatch, env, spec, u0, dt, steps=2, max_basis=30):
    """EPI2 through the phi-cycle JVP kernel selected by env=0 (strip / z-march) and env=1
    (the element-tile kernel, whose operator matches the oracle above)."""
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv(env, v)
        c = pkg.Context(0, fused=False)
        op = pkg.Operator(c, spec)
        out.append(pkg.integrate(c, op, to_dev(u0), "epi2", dt, steps * dt, tol=1e-10, max_basis=max_basis,
                                 orth_length=max_basis))
    return out


@pytest.mark.parametrize("order,nx,ny,periodic,flux", [
    (4, 40, 3, True, "ef"),    # one full 32-element strip + a partial one
    (4, 33, 4, False, "lf"),   # Dirichlet ends, a 1-element strip
    (7, 18, 3, True, "lf"),    # 16-element strips at order 7
    (2, 5, 6, False, "ef"),
])
def test_burgers2d_strip_matches_tile_kernel(monkeypatch, order, nx, ny, periodic, flux):
    rng = np.random.default_rng(7 * nx + order)
    spec = pkg.OperatorSpec("burgers2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), periodic=periodic, kappa=1e-2,
                            flux=flux, sigma=1e-3 if flux == "ef" else 0.0)
    u0 = 0.5 + 0.1 * rng.standard_normal(nx * ny * (order + 1) ** 2)
    a, b = _two_kernels(monkeypatch, "EXPDG_B2_TILE", spec, u0, 1e-3)
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)


@pytest.mark.parametrize("order,nx,ny,periodic,flux,fused", [
    (4, 64, 5, True, "ef", True),    # two full 32-element strips: the sweep takes the dots
    (4, 32, 4, False, "lf", True),   # Dirichlet ends
    (5, 32, 3, True, "lf", True),    # order 5: 6 V stages
    (7, 32, 3, True, "ef", True),    # 16-element strips at order 7
    (2, 32, 6, False, "ef", True),
    (4, 40, 3, True, "ef", False),   # a partial strip: the separate dots pass
])
def test_burgers2d_fused_dots_match_dots_pass(monkeypatch, order, nx, ny, periodic, flux, fused):
    # the 2D Burgers strip JVP takes the DCGS2 pass-1 dots of columns j <= 43 in its own sweep
    # on meshes of full strips (EXPDG_B2_DOTS=0: the separate k_ts2 dots pass)
    rng = np.random.default_rng(11 * nx + order)
    spec = pkg.OperatorSpec("burgers2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), periodic=periodic, kappa=1e-2,
                            flux=flux, sigma=1e-3 if flux == "ef" else 0.0)
    u0 = 0.5 + 0.1 * rng.standard_normal(nx * ny * (order + 1) ** 2)
    out = []
    for v in ("1", "0"):
        monkeypatch.setenv("EXPDG_B2_DOTS", v)
        c = pkg.Context(0, orth="dcgs2", fused=False, pipelined=False)  # the two-pass DCGS2's fused sweep
        op = pkg.Operator(c, spec)
        r = pkg.integrate(c, op, to_dev(u0), "epi2", 1e-3, 2e-3, tol=1e-10, max_basis=48, orth_length=48)
        r.alg_bytes = c.traffic()["alg_bytes"]
        out.append(r)
    a, b = out
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)
    if fused:
        assert a.alg_bytes < b.alg_bytes  # the sweep took the dots (u and w not re-read)
    else:
        assert a.alg_bytes == b.alg_bytes


def test_c3_fused_dots_epi2_parity():
    # C3 physics on 32^2 elements (full strips) through the fused JVP + DCGS2 dots sweep vs the oracle
    w = configs.scaled(configs.C3, 32, steps=3)
    u0 = w.initial_condition()
    orc = oracle_problem(w.spec()).integrate("epi2", u0, w.dt, w.steps * w.dt, tol=w.tol, max_basis=w.max_basis,
                                             orth_length=w.max_basis)
    c = pkg.Context(0, orth="dcgs2")
    op = pkg.Operator(c, w.spec())
    r = pkg.integrate(c, op, to_dev(u0), "epi2", w.dt, w.steps * w.dt, tol=w.tol, max_basis=w.max_basis,
                      orth_length=w.max_basis)
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    d_dev = np.diff(np.concatenate([[0], r.iters_per_step]))
    d_orc = np.diff(np.concatenate([[0], orc.iters_per_step]))
    assert np.max(np.abs(d_dev - d_orc)) <= 1


@pytest.mark.parametrize("order,dims", [(3, (3, 5, 4)), (3, (4, 4, 1)), (1, (5, 9, 3)), (1, (4, 8, 2))])
def test_euler3d_march_matches_tile_kernel(monkeypatch, order, dims):
    # odd meshes leave partial 2x2 (order 3) / 4x8 (order 1) tiles; nz = 1 wraps onto itself
    rng = np.random.default_rng(order + sum(dims))
    nx, ny, nz = dims
    spec = pkg.OperatorSpec("euler3d", order, nx, ny, nz, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    u0 = random_state5(rng, nx * ny * nz, (order + 1) ** 3)
    a, b = _two_kernels(monkeypatch, "EXPDG_E3_TILE", spec, u0, 2e-3)
    assert a.status == b.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert list(a.iters_per_step) == list(b.iters_per_step)
