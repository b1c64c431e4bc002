"""Shared helpers of the GPU parity tests (oracle = checker only)."""
import numpy as np


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_dev(x):
    import torch
    return torch.tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


def to_host(t):
    return t.detach().cpu().numpy()


def matrix_with_spectrum(rng, n, lo, hi, nonnormality):
    t = np.diag(rng.uniform(lo, hi, n)) + np.triu(nonnormality * rng.standard_normal((n, n)), 1)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return q @ t @ q.T


def oracle_problem(spec):
    import oracle
    return oracle.Problem(spec.kind, spec.order, spec.nx, spec.ny, spec.nz, box=spec.box, periodic=spec.periodic,
                          kappa=spec.kappa, flux=spec.flux, sigma=spec.sigma, sigma_adaptive=spec.sigma_adaptive,
                          gamma=spec.gamma, euler_flux=spec.euler_flux,
                          over_integrate=spec.over_integrate, grade_x=spec.grade_x, grade_y=spec.grade_y,
                          grade_z=spec.grade_z)
