"""The role-split (face-warp) JVP kernels against the single-role kernels they replace.

k_e2_phi_strip_fw (2D Euler strip, ops_euler2d.cu) and k_e3_phi_march_fw (3D Euler z-march,
ops_euler3d.cu) compute the same face fluxes (the reference's rhs_faces loop,
proj/src/euler.cpp:260-297) and the same volume / differentiation arithmetic as
k_e2_phi_strip<..,4,0> / k_e3_phi_march<..,0>, only on different warps and one row / plane ahead:
the EPI2 results must be IDENTICAL bit for bit (same operations in the same order per node), on
partial strips / tiles, every device order, both fluxes, single-row units and slab partitions.
EXPDG_E2_FW / EXPDG_E3_FW = 0 select the single-role kernels (read when the operator is built).
"""
import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from tests.gpu_util import to_dev, to_host
from tests.test_gpu_euler2d import random_state
from tests.test_gpu_extensions import random_state5
from tests.test_gpu_multirank import run_ranks
from paper_2011_01316_b200.partition import slab_ranges

pytestmark = pytest.mark.gpu


def _epi2(spec, u0, dt, steps, ctx=None, max_basis=12):
    # pipelined DCGS2: every column's lookahead application (stage 2) runs the plain JVP kernel
    c = ctx or pkg.Context(0, orth="dcgs2", fused=False)
    op = pkg.Operator(c, spec)
    r = pkg.integrate(c, op, to_dev(u0), "epi2", dt, steps * dt, tol=1e-10, max_basis=max_basis, orth_length=max_basis)
    return r, to_host(r.u), c.last_path()


def _both(monkeypatch, env, spec, u0, dt, steps=2):
    # the step residual through the element-tile kernel in both runs: the strip residual
    # (k_e2_phi_strip_fw<.., 2>) sums its face terms in another order than the tile kernel, and this
    # file pins the JVP kernels bit for bit (the residual kernels are pinned to the oracle in
    # test_gpu_euler2d.py / test_gpu_extensions.py and against each other below)
    monkeypatch.setenv("EXPDG_E2_RHS_TILE", "1")
    monkeypatch.setenv("EXPDG_E3_RHS_TILE", "1")
    out = []
    for v in ("1", "0"):
        monkeypatch.setenv(env, v)
        out.append(_epi2(spec, u0, dt, steps))
    (a, ua, pa), (b, ub, pb) = out
    assert a.status == b.status == "completed"
    assert pa["pipelined"] and pb["pipelined"]
    assert list(a.iters_per_step) == list(b.iters_per_step)
    assert np.array_equal(ua, ub), float(np.max(np.abs(ua - ub)))


@pytest.mark.parametrize("order,nx,ny,flux", [
    (4, 12, 7, "lf"),    # C4's order: two full 5-element strips and a 2-element one
    (4, 11, 1, "roe"),   # a single element row: every unit is one row, wrapped onto itself
    (4, 5, 9, "roe"),    # one full strip
    (1, 40, 3, "lf"),    # 32-element strips at order 1, a partial one
    (2, 9, 4, "roe"),
    (3, 8, 8, "lf"),     # 8 elements of 16 nodes fill the node warps exactly
    (5, 7, 3, "lf"),
    (7, 3, 4, "roe"),    # two elements per strip
    (8, 2, 3, "lf"),     # one element per strip
])
def test_strip_face_warp_bit_identical(monkeypatch, order, nx, ny, flux):
    rng = np.random.default_rng(100 * order + nx)
    spec = pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), euler_flux=flux)
    u0 = random_state(rng, nx * ny, (order + 1) ** 2)
    _both(monkeypatch, "EXPDG_E2_FW", spec, u0, 2e-4)


@pytest.mark.parametrize("order,dims", [
    (3, (4, 4, 5)),    # whole 2 x 2 tiles
    (3, (5, 3, 4)),    # partial tiles in x and y
    (3, (2, 2, 1)),    # one plane, wrapped onto itself
    (3, (1, 5, 3)),    # a one-element-wide mesh
    (1, (9, 10, 3)),   # order 1: 4 x 8 tiles, partial
    (1, (8, 16, 2)),   # order 1: whole tiles
])
def test_march_face_warps_bit_identical(monkeypatch, order, dims):
    nx, ny, nz = dims
    rng = np.random.default_rng(10 * order + nx + ny)
    spec = pkg.OperatorSpec("euler3d", order, nx, ny, nz, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    u0 = random_state5(rng, nx * ny * nz, (order + 1) ** 3)
    _both(monkeypatch, "EXPDG_E3_FW", spec, u0, 2e-4)


@pytest.mark.parametrize("kind,env", [("euler2d", "EXPDG_E2_FW"), ("euler3d", "EXPDG_E3_FW")])
def test_face_warps_on_slab_partitions_bit_identical(monkeypatch, kind, env):
    # halo rows / planes of the neighbouring rank enter through the producer and are read (and
    # released) by the face warps only; host-staged groups of 3 ranks, slabs of 1-2 layers
    rng = np.random.default_rng(5)
    if kind == "euler2d":
        spec = pkg.OperatorSpec("euler2d", 4, 7, 5, box=(0, 1, 0, 2, 0, 1), euler_flux="lf")
        u0 = random_state(rng, 7 * 5, 25)
        axis = spec.ny
    else:
        spec = pkg.OperatorSpec("euler3d", 3, 3, 4, 5, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
        u0 = random_state5(rng, 3 * 4 * 5, 64)
        axis = spec.nz
    layer = u0.size // axis
    ranges = slab_ranges(axis, 3)
    res = []
    monkeypatch.setenv("EXPDG_E2_RHS_TILE", "1")
    monkeypatch.setenv("EXPDG_E3_RHS_TILE", "1")
    for v in ("1", "0"):
        monkeypatch.setenv(env, v)

        def fn(r, c):
            part = pkg.OperatorSpec(**{**spec.__dict__, "part": ranges[r]})
            out = _epi2(part, u0[ranges[r][0] * layer:ranges[r][1] * layer], 2e-4, 2, ctx=c)
            return out[1], list(out[0].iters_per_step), out[0].status

        res.append(run_ranks(3, fn, orth="dcgs2"))
    for a, b in zip(*res):
        assert a[2] == b[2] == "completed"
        assert a[1] == b[1]
        assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("order,nx,ny,flux", [(4, 12, 7, "lf"), (4, 11, 1, "roe"), (1, 40, 3, "lf"), (2, 9, 4, "roe"),
                                              (3, 8, 8, "lf"), (5, 7, 3, "roe"), (7, 3, 4, "lf"), (8, 2, 3, "roe")])
def test_strip_residual_matches_tile_kernel(monkeypatch, order, nx, ny, flux):
    # R(x) and the frozen primitives it leaves for the JVPs: the strip kernel (MODE 2, face warps)
    # against the element-tile kernel, through full_rhs and through one EPI2 step
    rng = np.random.default_rng(10 * order + nx)
    spec = pkg.OperatorSpec("euler2d", order, nx, ny, box=(0, 1, 0, 2, 0, 1), euler_flux=flux)
    u0 = random_state(rng, nx * ny, (order + 1) ** 2)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("EXPDG_E2_RHS_TILE", v)
        c = pkg.Context(0, orth="dcgs2", fused=False)
        op = pkg.Operator(c, spec)
        rhs = to_host(op.full_rhs(to_dev(u0)))
        op.linearize(to_dev(u0))
        x = 1.0 + 0.1 * np.cos(np.arange(u0.size))
        nl = to_host(op.apply_nonlinear(to_dev(u0 * x)))  # MODE 1: N at a state away from the frozen one
        r = pkg.integrate(c, op, to_dev(u0), "exprb32", 2e-4, 4e-4, tol=1e-10, max_basis=12, orth_length=12)
        out.append((rhs, to_host(r.u), list(r.iters_per_step), r.status, nl))
    (ra, ua, ia, sa, na), (rb, ub, ib, sb, nb) = out
    assert sa == sb == "completed" and ia == ib
    assert np.max(np.abs(ra - rb)) <= 1e-13 * np.max(np.abs(rb))
    assert np.max(np.abs(na - nb)) <= 1e-13 * np.max(np.abs(rb))
    assert np.max(np.abs(ua - ub)) <= 1e-13 * np.max(np.abs(ub))


@pytest.mark.parametrize("order,dims", [(3, (4, 4, 5)), (3, (5, 3, 4)), (3, (2, 2, 1)), (1, (9, 10, 3)), (1, (8, 16, 2))])
def test_march_residual_matches_tile_kernel(monkeypatch, order, dims):
    # the 3D counterpart: k_e3_phi_march_fw<.., 2> against k_e3_apply (mode 2)
    nx, ny, nz = dims
    rng = np.random.default_rng(order + nx + nz)
    spec = pkg.OperatorSpec("euler3d", order, nx, ny, nz, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
    u0 = random_state5(rng, nx * ny * nz, (order + 1) ** 3)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("EXPDG_E3_RHS_TILE", v)
        c = pkg.Context(0, orth="dcgs2", fused=False)
        op = pkg.Operator(c, spec)
        rhs = to_host(op.full_rhs(to_dev(u0)))
        op.linearize(to_dev(u0))
        x = 1.0 + 0.1 * np.cos(np.arange(u0.size))
        nl = to_host(op.apply_nonlinear(to_dev(u0 * x)))  # MODE 1: N at a state away from the frozen one
        r = pkg.integrate(c, op, to_dev(u0), "exprb32", 2e-4, 4e-4, tol=1e-10, max_basis=12, orth_length=12)
        out.append((rhs, to_host(r.u), list(r.iters_per_step), r.status, nl))
    (ra, ua, ia, sa, na), (rb, ub, ib, sb, nb) = out
    assert sa == sb == "completed" and ia == ib
    assert np.max(np.abs(ra - rb)) <= 1e-13 * np.max(np.abs(rb))
    assert np.max(np.abs(na - nb)) <= 1e-13 * np.max(np.abs(rb))
    assert np.max(np.abs(ua - ub)) <= 1e-13 * np.max(np.abs(ub))


@pytest.mark.parametrize("kind", ["euler2d", "euler3d"])
def test_strip_residual_reports_inadmissible_state(kind):
    # a negative density reaches the domain flag through the MODE 2 kernels like through the tile
    # kernels: integrate turns it into blew_up (proj/src/integrators.cpp:179-193)
    rng = np.random.default_rng(2)
    if kind == "euler2d":
        spec = pkg.OperatorSpec("euler2d", 4, 7, 3, box=(0, 1, 0, 2, 0, 1), euler_flux="lf")
        u0 = random_state(rng, 21, 25)
    else:
        spec = pkg.OperatorSpec("euler3d", 3, 3, 2, 3, box=(0, 1, 0, 2, 0, 1.5), euler_flux="lf")
        u0 = random_state5(rng, 18, 64)
    c = pkg.Context(0, fused=False)
    op = pkg.Operator(c, spec)
    good = pkg.integrate(c, op, to_dev(u0), "epi2", 2e-4, 2e-4, tol=1e-10, max_basis=12, orth_length=12)
    assert good.status == "completed"
    u0[7] = -1.0  # density of node 7 of element 0
    bad = pkg.integrate(c, op, to_dev(u0), "epi2", 2e-4, 2e-4, tol=1e-10, max_basis=12, orth_length=12)
    assert bad.status == "blew_up" and bad.blow_up_step == 1
