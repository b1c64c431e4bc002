"""GPU parity: device phi engine (proj/src/phi.cpp) on the reference's dense fakes
(proj/tests/test_phi.cpp, acceptance criterion 1) against the oracle."""
import math

import numpy as np
import pytest

import oracle
import paper_2011_01316_b200 as pkg
from tests.gpu_util import matrix_with_spectrum, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return pkg.Context(0)


def test_dense_fake_matches_dense_oracle(ctx):
    # proj/tests/test_phi.cpp:209-230
    rng = np.random.default_rng(2024)
    n = 50
    M = matrix_with_spectrum(rng, n, -20.0, 1.0, 1.0)
    b = [rng.standard_normal(n) for _ in range(4)]
    dt = 0.7
    fam = oracle.phi_dense_family(3, dt * M)
    expect = sum(dt ** i * fam[i] @ b[i] for i in range(4))
    op = pkg.Operator(ctx, dense=M)
    got, st = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], dt, tol=1e-10)
    assert rel(to_host(got), expect) < 1e-8
    ref, iters, subs = oracle.phi_combination_dense(M, b, dt, tol=1e-10)
    assert rel(to_host(got), ref) < 1e-10
    assert abs(st.iterations - iters) <= 1 and st.substeps == subs


def test_criterion1_random_cases(ctx):
    # acceptance criterion 1 (proj/tests/acceptance.cpp:70-108): worst dev <= 1e-8
    rng = np.random.default_rng(20240601)
    worst = 0.0
    for trial in range(30):
        n = int(rng.integers(10, 101))
        M = matrix_with_spectrum(rng, n, -50.0, 2.0, 1.0)
        b = [rng.standard_normal(n) for _ in range(4)]
        fam = oracle.phi_dense_family(3, M)
        expect = sum(fam[i] @ b[i] for i in range(4))
        op = pkg.Operator(ctx, dense=M)
        got, _ = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], 1.0, tol=1e-10)
        worst = max(worst, rel(to_host(got), expect))
    assert worst <= 1e-8


def test_trivial_cases(ctx):
    # proj/tests/test_phi.cpp:166-207
    rng = np.random.default_rng(5)
    n = 8
    op = pkg.Operator(ctx, dense=np.zeros((n, n)))
    b0 = rng.standard_normal(n)
    got, _ = pkg.phi_combination(ctx, op, [to_dev(b0)], 0.3)
    assert np.abs(to_host(got) - b0).max() < 1e-13
    bs = [rng.standard_normal(n) for _ in range(4)]
    got, _ = pkg.phi_combination(ctx, op, [to_dev(v) for v in bs], 0.7)
    expect = sum(0.7 ** i / math.factorial(i) * bs[i] for i in range(4))
    assert np.abs(to_host(got) - expect).max() < 1e-12
    got, _ = pkg.phi_combination(ctx, op, [to_dev(np.zeros(n)), to_dev(np.zeros(n))], 1.0)
    assert np.linalg.norm(to_host(got)) == 0.0


def test_iop_window_matches_oracle(ctx):
    rng = np.random.default_rng(3)
    n = 80
    M = matrix_with_spectrum(rng, n, -30.0, 0.5, 0.5)
    b = [np.zeros(n), rng.standard_normal(n)]
    op = pkg.Operator(ctx, dense=M)
    got, st = pkg.phi_combination(ctx, op, [to_dev(v) for v in b], 1.0, tol=1e-10, max_basis=40, orth_length=4)
    ref, iters, subs = oracle.phi_combination_dense(M, b, 1.0, tol=1e-10, max_basis=40, orth_length=4)
    assert rel(to_host(got), ref) < 1e-9
    assert abs(st.iterations - iters) <= 1


def test_semigroup_and_linearity(ctx):
    rng = np.random.default_rng(31)
    n = 40
    M = matrix_with_spectrum(rng, n, -15.0, 0.5, 1.0)
    op = pkg.Operator(ctx, dense=M)
    b0 = rng.standard_normal(n)
    whole, _ = pkg.phi_combination(ctx, op, [to_dev(b0)], 1.0, tol=1e-12)
    half, _ = pkg.phi_combination(ctx, op, [to_dev(b0)], 0.5, tol=1e-12)
    chained, _ = pkg.phi_combination(ctx, op, [half.clone()], 0.5, tol=1e-12)
    assert rel(to_host(chained), to_host(whole)) < 1e-11


def test_krylov_error_budget(ctx):
    # a stiff operator with a 1-substep budget raises KrylovError (proj/src/phi.cpp:186-188)
    rng = np.random.default_rng(8)
    n = 60
    M = matrix_with_spectrum(rng, n, -5000.0, 0.0, 1.0)
    op = pkg.Operator(ctx, dense=M)
    with pytest.raises(pkg.KrylovError):
        pkg.phi_combination(ctx, op, [None, to_dev(rng.standard_normal(n))], 1.0, tol=1e-12, max_basis=8,
                            max_substeps=1)


@pytest.mark.parametrize("n", [1, 2, 7, 17, 42, 105, 130])
def test_device_expm_matches_oracle(ctx, n):
    # the controller's expm (csrc/ctl.cuh blk_expm: Higham 2005 scaling and squaring, Pade
    # 3/5/7/9/13) through the exported expdg_expm, against the oracle's restatement of the
    # Eigen MatrixFunctions exp() the reference calls (proj/src/phi.cpp:40), over 1-norms
    # 1e-3 .. 300 (every Pade degree and squaring counts 0 .. 9)
    rng = np.random.default_rng(1000 + n)
    worst = 0.0
    for norm in (1e-3, 1e-1, 0.5, 2.0, 5.0, 20.0, 80.0, 300.0):
        # Hessenberg-like (the controller's input) and dense non-normal, negative-heavy spectra
        for shape in ("hess", "dense"):
            A = rng.standard_normal((n, n))
            if shape == "hess":
                A = np.triu(A, -1)
            A -= 0.5 * np.abs(np.diag(np.diag(A))) * (shape == "dense")
            A *= norm / max(np.abs(A).sum(axis=0).max(), 1e-300)
            got = ctx.expm(A)
            ref = oracle.expm(A)
            assert np.all(np.isfinite(got))
            worst = max(worst, rel(got, ref))
    assert worst <= 1e-12, worst
