"""Reference-file / CSV formats of the reference harness (proj/src/harness.cpp:240-353,
:481-495), restated in paper_2011_01316_b200/refio.py (host-side, CPU)."""
import math

import numpy as np
import pytest

import oracle
from paper_2011_01316_b200 import refio


def test_filename_matches_reference_rules():
    s = refio.ReferenceSpec("burgers-smooth", "lf", over_integrate=True, kappa=0.03, integrator="rk4", k=4, ne=40,
                            dt=1e-5, t_final=1.0)
    assert refio.reference_filename(s) == "burgers-smooth_lf_oi_kap0.03_rk4_k4_ne40_dt1e-05_t1.ref"
    s2 = refio.ReferenceSpec("burgers-mms", "ef", sigma=3e-4, kappa=0.01, k=6, ne=80, dt=2.5e-6, t_final=0.01)
    assert refio.reference_filename(s2) == "burgers-mms_ef_s0.0003_kap0.01_rk4_k6_ne80_dt2.5e-06_t0.01.ref"
    s3 = refio.ReferenceSpec("burgers-smooth", "ef", sigma=1.0, sigma_adaptive=True)
    assert "_sadapt_" in refio.reference_filename(s3) and "_s1_" not in refio.reference_filename(s3)


def test_round_trip_and_header(tmp_path):
    s = refio.ReferenceSpec("burgers-smooth", "lf", over_integrate=True, k=3, ne=20, dt=1e-5, t_final=1.0)
    u = oracle.rk4_reference("burgers-smooth", 20, 3, "lf", 1, 1e-3, 0.05)
    path = str(tmp_path / refio.reference_filename(s))
    refio.save_reference(path, s, u)
    lines = open(path).read().split("\n")
    assert lines[:15] == ["expdg-reference-v1", "problem burgers-smooth", "flux lf", "sigma 0", "sigma_adaptive 0",
                          "over_integrate 1", "kappa 0.029999999999999999", "integrator rk4", "k 3", "ne 20",
                          "dt 1.0000000000000001e-05", "t_final 1", "components 1", "size 80", lines[14]]
    assert float(lines[14]) == u[0]
    back = refio.load_reference(path, s)
    assert np.array_equal(back, u)  # %.17g round-trips doubles exactly


def test_metadata_mismatch_and_truncation(tmp_path):
    s = refio.ReferenceSpec("burgers-smooth", k=2, ne=4)
    path = str(tmp_path / "r.ref")
    refio.save_reference(path, s, np.arange(12.0))
    for field, value in [("kappa", 0.02), ("k", 3), ("integrator", "rk2"), ("flux", "ef"), ("dt", 2e-5)]:
        bad = refio.ReferenceSpec(**{**s.__dict__, field: value})
        with pytest.raises(RuntimeError):
            refio.load_reference(path, bad)
    txt = open(path).read().rsplit("\n", 3)[0] + "\n"
    open(path, "w").write(txt)
    with pytest.raises(RuntimeError):
        refio.load_reference(path, s)


def test_experiment_csv_layout():
    rows = [refio.ExperimentRow(0.1, [1e-3, float("nan")], [float("nan"), 2.0], 0.5, 3.25, 17, 0.125, "completed")]
    csv = refio.experiment_csv(rows, ["rho", "rhou"])
    head, row, _ = csv.split("\n")
    assert head == "scale,error_rho,error_rhou,order_rho,order_rhou,cr_a,cr_d,krylov_iters,wallclock_s,status"
    assert row == "0.10000000000000001,0.001,,,2,0.5,3.25,17,0.125,completed"
