"""GPU parity of the EXACT engine path bench.py times, against the oracle.

The bench runs AUTO orthogonalisation, which selects DCGS2 by size (n >= 2^18 DOF,
csrc/krylov.cu Engine::config), with the operator sweep taking the DCGS2 pass-1 dots
(`k_e2_phi_strip<..,DOT>`, `k_b2_phi_strip<..,DOT>`, `k_e3_phi_march<..,DOT>`) and
device-resident control in CUDA-graph WHILE nodes.  These tests run that path — selected
by size, not forced — on meshes just large enough to trigger it, and compare with the
oracle (the CPU restatement of proj/src/phi.cpp:84-112, :133-260 with its MGS2 Arnoldi):
relative L2 <= 1e-9 after the final step and Krylov dimensions per step equal +-1 (the
north star's bar).  `ctx.last_path()` proves which path ran.
"""
import numpy as np
import pytest

import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


def _dims(r):
    return np.diff(np.concatenate([[0], np.asarray(r.iters_per_step)]))


def _run_both(w, steps, integrator="epi2", pipelined=None):
    ctx = pkg.Context(0, pipelined=pipelined)  # AUTO orthogonalisation (the bench's context)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    op = pkg.Operator(ctx, w.spec())
    r = pkg.integrate(ctx, op, to_dev(u0), integrator, dt, steps * dt, **kw)
    path = ctx.last_path()
    orc = oracle_problem(w.spec()).integrate(integrator, u0, dt, steps * dt, **kw)
    return r, orc, path, op.dim


@pytest.mark.parametrize("pipelined", [True, False])
@pytest.mark.parametrize("name,nx,steps", [
    ("C4", 64, 5),    # 2D Euler vortex, 409,600 DOF: DCGS2 + fused strip dots (the bench workload's path)
    ("C3", 128, 5),   # 2D Burgers, 409,600 DOF, nx % 32 == 0: DCGS2 + fused strip dots
    ("C5", 16, 3),    # 3D Euler TGV, 1,310,720 DOF, whole 2x2 tiles: DCGS2 + fused z-march dots
])
def test_bench_path_matches_oracle(name, nx, steps, pipelined):
    # pipelined (the default): one basis stream per column (k_ts3) after a lookahead application;
    # the fused sweep dots then serve the first column of every substep
    w = configs.scaled(configs.ALL[name], nx, steps=steps)
    r, orc, path, n = _run_both(w, steps, pipelined=pipelined)
    assert n >= 1 << 18
    assert path == {"dcgs2": True, "pipelined": pipelined, "fused_dots": True, "graph": True,
                    "fused_engine": False}, path
    assert r.status == orc.status == "completed"
    assert r.steps == orc.steps == steps
    err = rel(to_host(r.u), orc.u)
    assert err <= 1e-9, err
    d_dev, d_orc = _dims(r), _dims(orc)
    print(f"{name}@{nx} pipelined={pipelined}: n={n} rel L2 {err:.3e}, Krylov dims device {d_dev.tolist()} oracle {d_orc.tolist()}")
    assert len(d_dev) == len(d_orc) == steps
    assert np.max(np.abs(d_dev - d_orc)) <= 1, (d_dev, d_orc)


def test_c4_bench_path_host_stepped_matches_graph():
    # the bench's roofline leg re-runs one step host-stepped (use_graph = False): same kernels,
    # so the same bits as the graph-controlled step
    w = configs.scaled(configs.C4, 64, steps=1)
    ctx = pkg.Context(0)
    u0 = w.initial_condition()
    dt = w.time_step(u0)
    op = pkg.Operator(ctx, w.spec())
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    a = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, dt, **kw)
    b = pkg.integrate(ctx, op, to_dev(u0), "epi2", dt, dt, use_graph=False, **kw)
    assert ctx.last_path()["graph"] is False and ctx.last_path()["fused_dots"] is True
    assert np.array_equal(to_host(a.u), to_host(b.u))
    assert a.krylov_iterations == b.krylov_iterations


@pytest.mark.slow
def test_c4_full_size_one_step_matches_oracle():
    # EXPDG_SLOW=1: the bench workload itself (C4, 1024^2, 104,857,600 DOF), one EPI2 step,
    # device vs the oracle on the GPU box's host (~35 GB of oracle Krylov basis, minutes)
    w = configs.C4
    r, orc, path, n = _run_both(w, 1)
    assert path["dcgs2"] and path["fused_dots"] and path["graph"]
    assert r.status == orc.status == "completed"
    err = rel(to_host(r.u), orc.u)
    print(f"C4 1024^2: rel L2 {err:.3e}, Krylov iterations device {r.krylov_iterations} oracle "
          f"{orc.krylov_iterations}, oracle {orc.seconds:.0f} s")
    assert err <= 1e-9
    assert abs(int(r.krylov_iterations) - int(orc.krylov_iterations)) <= 1


def test_exprb42_on_pipelined_path_matches_oracle():
    # the p = 3 phi calls of EXPRB42 (proj/src/integrators.cpp:100-113) on the pipelined DCGS2 path
    w = configs.scaled(configs.C4, 64, steps=2)
    r, orc, path, n = _run_both(w, 2, integrator="exprb42")
    assert path["pipelined"] and path["graph"]
    assert r.status == orc.status == "completed"
    assert rel(to_host(r.u), orc.u) <= 1e-9
    assert np.max(np.abs(_dims(r) - _dims(orc))) <= 1


def test_user_operator_on_pipelined_path_matches_oracle():
    # a user LinearAction at n >= 2^18 DOF: AUTO selects the pipelined DCGS2, whose lookahead
    # application calls the user's action on slot j+1 (tests/test_gpu_user_op.py's split, larger)
    import math

    import oracle
    import torch
    n = 1 << 18
    h = 2 * math.pi / n
    x = np.arange(n) * h
    ref = 0.5 + np.sin(x)
    nu = 1e-6

    def L_np(v):
        return -(np.roll(ref * v, -1) - np.roll(ref * v, 1)) / (2 * h) + nu * (np.roll(v, -1) - 2 * v + np.roll(v, 1)) / h ** 2

    rt = torch.tensor(ref, device="cuda:0")

    def L_t(v):
        return -(torch.roll(rt * v, -1) - torch.roll(rt * v, 1)) / (2 * h) + nu * (torch.roll(v, -1) - 2 * v + torch.roll(v, 1)) / h ** 2

    rng = np.random.default_rng(3)
    b = [rng.standard_normal(n), np.sin(3 * x)]
    dt = 2e-5
    ctx = pkg.Context(0)
    op = pkg.UserOperator(ctx, pkg.SplitProblem(n, linear=L_t))
    got, st = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], dt, tol=1e-10, max_basis=40, orth_length=40)
    path = ctx.last_path()
    assert path["pipelined"], path
    exp_, iters, subs = oracle.phi_combination_user(L_np, n, b, dt, tol=1e-10, max_basis=40, orth_length=40)
    assert rel(to_host(got), exp_) <= 1e-10
    assert abs(st.iterations - iters) <= 1 and st.substeps == subs
