"""GPU: the fused single-CTA engine for small problems (csrc/fused.cuh) against the
multi-kernel engine and the oracle — same algorithm, so same Krylov dimensions."""
import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
from tests.gpu_util import oracle_problem, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("integ", ["epi2", "exprb42", "exp_euler"])
def test_fused_matches_multikernel_and_oracle(integ):
    w = configs.scaled(configs.C1_S3E4, 128, steps=20)
    u0 = w.initial_condition()
    kw = dict(tol=w.tol, max_basis=30, orth_length=30)
    res = {}
    for fused in (True, False):
        ctx = pkg.Context(0, fused=fused)
        res[fused] = pkg.integrate(ctx, pkg.Operator(ctx, w.spec()), to_dev(u0), integ, w.dt, w.steps * w.dt, **kw)
        if fused:
            assert ctx.kernel_launches < 20 * 20  # a handful of kernels per step, not ~6 per Krylov column
    orc = oracle_problem(w.spec()).integrate(integ, u0, w.dt, w.steps * w.dt, **kw)
    a, b = res[True], res[False]
    assert a.status == b.status == orc.status == "completed"
    assert rel(to_host(a.u), to_host(b.u)) <= 1e-12
    assert rel(to_host(a.u), orc.u) <= 1e-9
    assert np.max(np.abs(np.diff(np.concatenate([[0], a.iters_per_step])) -
                         np.diff(np.concatenate([[0], orc.iters_per_step])))) <= 1


def test_fused_iop_window_and_phi_api():
    # IOP window (orth_length < max_basis) and the phi_combination entry point
    w = configs.scaled(configs.C1_S3E4, 96, steps=1)
    u0 = w.initial_condition()
    spec = w.spec()
    orc = oracle_problem(spec)
    r = orc.apply_linear(u0, u0) + orc.apply_nonlinear(u0, u0)
    outs = []
    for fused in (True, False):
        ctx = pkg.Context(0, fused=fused)
        op = pkg.Operator(ctx, spec)
        op.linearize(to_dev(u0))
        out, st = pkg.phi_combination(ctx, op, [None, to_dev(r)], 0.02, tol=1e-10, max_basis=30, orth_length=4)
        outs.append((to_host(out), st.iterations, st.substeps))
    assert rel(outs[0][0], outs[1][0]) <= 1e-12
    assert outs[0][1:] == outs[1][1:]
