"""ORACLE — test infrastructure only (see oracle/include/oracle.hpp).

ctypes bindings for the Eigen-free CPU restatement of the reference library
(/root/reference/proj).  Importable only from tests/, __graft_entry__.smoke()
and bench.py's CPU legs, where it is the checker / the CPU baseline — never the
thing measured on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None
# user LinearAction / SplitProblem callbacks on host vectors: (x, y, user) -> status, (ref, user) -> status
USER_APPLY = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)
USER_LINEARIZE = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_void_p)


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (outputs only under oracle/_build)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    else:
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class ProblemDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("order", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("z0", C.c_double), ("z1", C.c_double),
        ("bc", C.c_int), ("kappa", C.c_double), ("flux", C.c_int), ("sigma", C.c_double),
        ("sigma_adaptive", C.c_int), ("over_integrate", C.c_int),
        ("gamma", C.c_double), ("euler_flux", C.c_int),
        ("grade_x", C.POINTER(C.c_double)), ("grade_y", C.POINTER(C.c_double)), ("grade_z", C.POINTER(C.c_double)),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_problem_create.restype = C.c_void_p
        L.oracle_problem_create.argtypes = [C.POINTER(ProblemDesc)]
        L.oracle_problem_destroy.argtypes = [C.c_void_p]
        L.oracle_problem_dim.restype = C.c_long
        L.oracle_problem_dim.argtypes = [C.c_void_p]
        L.oracle_apply.argtypes = [C.c_void_p, C.c_int, dp, dp, dp]
        L.oracle_burgers_diag.argtypes = [C.c_void_p, dp, dp, dp, dp, dp, dp, dp]
        L.oracle_burgers_inner.argtypes = [C.c_void_p, dp, dp, dp]
        L.oracle_integrate.argtypes = [C.c_void_p, C.c_int, dp, C.c_double, C.c_double, C.c_double,
                                       C.c_int, C.c_int, C.c_int, C.POINTER(C.c_long), dp,
                                       C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       dp, C.POINTER(C.c_long), dp, C.c_int, dp, dp, C.c_int,
                                       C.POINTER(C.c_int)]
        L.oracle_phi_user.argtypes = [C.c_int, USER_APPLY, C.c_void_p, C.c_int, dp, C.c_double, C.c_double,
                                      C.c_int, C.c_int, dp, C.POINTER(C.c_long), C.POINTER(C.c_int), dp]
        L.oracle_integrate_user.argtypes = [C.c_long, USER_APPLY, USER_APPLY, USER_LINEARIZE, C.c_void_p, C.c_int,
                                            dp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(C.c_long), dp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), dp, C.POINTER(C.c_long), C.c_int, dp, dp,
                                            C.c_int, C.POINTER(C.c_int)]
        L.oracle_phi_dense_op.argtypes = [C.c_int, dp, C.c_int, dp, C.c_double, C.c_double, C.c_int,
                                          C.c_int, dp, C.POINTER(C.c_long), C.POINTER(C.c_int), dp]
        L.oracle_expm.argtypes = [C.c_int, dp, dp]
        L.oracle_phi_dense_family.argtypes = [C.c_int, C.c_int, dp, dp]
        L.oracle_phi_scalar.restype = C.c_double
        L.oracle_phi_scalar.argtypes = [C.c_int, C.c_double]
        L.oracle_krylov_build.argtypes = [C.c_int, dp, dp, C.c_int, C.c_int, dp, dp,
                                          C.POINTER(C.c_int), C.POINTER(C.c_int), dp]
        L.oracle_lgl.argtypes = [C.c_int, dp, dp, dp]
        L.oracle_gauss.argtypes = [C.c_int, dp, dp]
        L.oracle_euler_pointwise.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, C.c_double, dp]
        L.oracle_burgers_flux.restype = C.c_double
        L.oracle_burgers_flux.argtypes = [C.c_int] + [C.c_double] * 5
        L.oracle_vortex.argtypes = [C.c_double, C.c_double, C.c_double, dp, C.c_double, dp]
        L.oracle_ic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, dp]
        L.oracle_splitmix_normal.restype = C.c_double
        L.oracle_splitmix_normal.argtypes = [C.c_uint64, C.c_int, dp]
        L.oracle_courant.argtypes = [C.c_void_p, dp, C.c_double, dp, dp]
        L.oracle_acc_mms.argtypes = [C.c_int, C.c_int, C.c_double, dp]
        L.oracle_acc_temporal.argtypes = [C.c_int, dp]
        L.oracle_acc_large_courant.argtypes = [dp]
        L.oracle_acc_vortex.argtypes = [C.c_int, dp]
        L.oracle_acc_burgers_order.restype = C.c_double
        L.oracle_acc_burgers_order.argtypes = [C.c_int]
        L.oracle_acc_ode_order.restype = C.c_double
        L.oracle_acc_ode_order.argtypes = [C.c_int]
        L.oracle_acc_exp_euler_joint.argtypes = [dp]
        L.oracle_harness_burgers.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_double, C.c_int,
                                             C.c_int, C.c_double, dp, dp, dp]
        L.oracle_l2_error_exact.restype = C.c_double
        L.oracle_mms_source.restype = C.c_double
        L.oracle_mms_source.argtypes = [C.c_double, C.c_double]
        L.oracle_l2_error_exact.argtypes = [C.c_char_p, C.c_int, C.c_int, dp, C.c_double, C.c_int]
        L.oracle_harness_u0.restype = C.c_long
        L.oracle_harness_u0.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p]
        L.oracle_rk4_reference.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_double,
                                           C.c_double, dp]
        L.oracle_l2_error_discrete.restype = C.c_double
        L.oracle_l2_error_discrete.argtypes = [C.c_char_p, C.c_int, C.c_int, dp, C.c_int, C.c_int, dp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class OracleError(RuntimeError):
    pass


class KrylovError(OracleError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise ArithmeticError(msg)
    if rc == 4:
        raise KrylovError(msg)
    raise OracleError(msg)


INTEGRATORS = {"exp_euler": 0, "epi2": 1, "exprb32": 2, "exprb42": 3, "rk2": 4, "rk3": 5, "rk4": 6}


@dataclass
class IntegrationResult:
    u: np.ndarray
    steps: int
    status: str
    blow_up_step: int
    max_abs: float
    krylov_iterations: int
    iters_per_step: np.ndarray  # cumulative, per completed step
    amax_per_step: np.ndarray
    seconds: float
    snapshots: list = None


class Problem:
    """An oracle problem (mesh + basis + operator config)."""

    KINDS = {"burgers1d": 1, "burgers2d": 2, "euler2d": 3, "euler3d": 4}

    def __init__(self, kind: str, order: int, nx: int, ny: int = 1, nz: int = 1,
                 box=(0.0, 1.0, 0.0, 1.0, 0.0, 1.0), periodic: bool = True, kappa: float = 0.03,
                 flux: str = "lf", sigma: float = 0.0, sigma_adaptive: bool = False,
                 over_integrate: bool = False, gamma: float = 1.4, euler_flux: str = "lf",
                 grade_x=None, grade_y=None, grade_z=None):
        d = ProblemDesc()
        d.kind = self.KINDS[kind]
        d.order, d.nx, d.ny, d.nz = order, nx, ny, nz
        d.x0, d.x1, d.y0, d.y1, d.z0, d.z1 = box
        d.bc = 0 if periodic else 1
        d.kappa, d.flux, d.sigma = kappa, (1 if flux in ("ef", "entropy") else 0), sigma
        d.sigma_adaptive, d.over_integrate = int(sigma_adaptive), int(over_integrate)
        d.gamma, d.euler_flux = gamma, (0 if euler_flux == "roe" else 1)
        # grading lists (proj/src/mesh.cpp:96-120): kept alive with the problem
        self._grades = [None if g is None else np.ascontiguousarray(g, dtype=np.float64)
                        for g in (grade_x, grade_y, grade_z)]
        d.grade_x, d.grade_y, d.grade_z = [None if g is None else _p(g) for g in self._grades]
        self.desc = d
        self.kind = kind
        self.h = lib().oracle_problem_create(C.byref(d))
        if not self.h:
            raise ValueError(lib().oracle_last_error().decode())
        self.dim = lib().oracle_problem_dim(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_problem_destroy(self.h)
            self.h = None

    def _apply(self, which, ref, x):
        ref = np.ascontiguousarray(ref if ref is not None else np.zeros(self.dim), dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.dim)
        _check(lib().oracle_apply(self.h, which, _p(ref), _p(x), _p(y)))
        return y

    def apply_linear(self, ref, x):
        return self._apply(0, ref, x)

    def apply_nonlinear(self, ref, x):
        return self._apply(1, ref, x)

    def full_rhs(self, x):
        return self._apply(2, None, x)

    def courant(self, u, dt):
        a, d = C.c_double(), C.c_double()
        u = np.ascontiguousarray(u, dtype=np.float64)
        lib().oracle_courant(self.h, _p(u), dt, C.byref(a), C.byref(d))
        return a.value, d.value

    def integrate(self, integrator: str, u0, dt, t_final, tol=1e-12, max_basis=128,
                  orth_length=128, max_steps=None, snapshot_every=0) -> IntegrationResult:
        u = np.array(u0, dtype=np.float64, copy=True)
        nsteps_cap = max_steps or int(np.ceil(t_final / dt + 1e-9)) + 2
        iters = np.zeros(nsteps_cap, dtype=np.int64)
        amax = np.zeros(nsteps_cap)
        steps, status, bus = C.c_int(), C.c_int(), C.c_int()
        mx, tot, secs = C.c_double(), C.c_long(), C.c_double()
        scap = nsteps_cap // snapshot_every if snapshot_every > 0 else 0
        snaps, snap_t, nsn = np.zeros((max(scap, 1), self.dim)), np.zeros(max(scap, 1)), C.c_int()
        _check(lib().oracle_integrate(self.h, INTEGRATORS[integrator], _p(u), dt, t_final, tol,
                                      max_basis, orth_length, nsteps_cap,
                                      iters.ctypes.data_as(C.POINTER(C.c_long)), _p(amax),
                                      C.byref(steps), C.byref(status), C.byref(bus), C.byref(mx),
                                      C.byref(tot), C.byref(secs), snapshot_every, _p(snaps), _p(snap_t),
                                      scap, C.byref(nsn)))
        n_ok = steps.value if status.value == 0 else steps.value - 1
        res = IntegrationResult(u, steps.value, "completed" if status.value == 0 else "blew_up",
                                bus.value, mx.value, tot.value, iters[:n_ok].copy(),
                                amax[:n_ok].copy(), secs.value)
        res.snapshots = [(float(snap_t[k]), snaps[k].copy()) for k in range(min(nsn.value, scap))]
        return res


def _user_apply(f, n):
    def cb(x, y, _user):
        try:
            out = f(np.ctypeslib.as_array(x, (n,)).copy())
            np.ctypeslib.as_array(y, (n,))[:] = out
            return 0
        except ArithmeticError:
            return 2
        except ValueError:
            return 1
    return USER_APPLY(cb)


def phi_combination_user(apply, n, b_list, dt, tol=1e-12, max_basis=128, orth_length=128):
    """phi_combination (proj/src/phi.cpp:133-260) with a user LinearAction `apply(x) -> y` (numpy)."""
    cb = _user_apply(apply, n)
    b = np.ascontiguousarray(np.stack(b_list), dtype=np.float64)
    out = np.empty(n)
    iters, subs, est = C.c_long(), C.c_int(), C.c_double()
    _check(lib().oracle_phi_user(n, cb, None, len(b_list) - 1, _p(b), dt, tol, max_basis, orth_length,
                                 _p(out), C.byref(iters), C.byref(subs), C.byref(est)))
    return out, iters.value, subs.value


def integrate_user(n, linearize, integrator, u0, dt, t_final, tol=1e-12, max_basis=128, orth_length=128,
                   snapshot_every=0) -> IntegrationResult:
    """integrate (proj/src/integrators.cpp:140-201) of a user SplitProblem: `linearize(ref)` returns
    (linear, nonlinear) callables on numpy vectors (nonlinear may be None)."""
    state = {}

    def lin_cb(ref, _user):
        try:
            L, N = linearize(np.ctypeslib.as_array(ref, (n,)).copy())
            state["L"], state["N"] = L, N
            return 0
        except ArithmeticError:
            return 2
        except ValueError:
            return 1

    a_l = _user_apply(lambda x: state["L"](x), n)
    a_n = _user_apply(lambda x: state["N"](x) if state["N"] is not None else np.zeros(n), n)
    c_lin = USER_LINEARIZE(lin_cb)
    u = np.array(u0, dtype=np.float64, copy=True)
    cap = int(np.ceil(t_final / dt + 1e-9)) + 2
    iters = np.zeros(cap, dtype=np.int64)
    amax = np.zeros(cap)
    steps, status, bus, nsn = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    mx, tot = C.c_double(), C.c_long()
    scap = cap // snapshot_every if snapshot_every > 0 else 0
    snaps, snap_t = np.zeros((max(scap, 1), n)), np.zeros(max(scap, 1))
    _check(lib().oracle_integrate_user(n, a_l, a_n, c_lin, None, INTEGRATORS[integrator], _p(u), dt, t_final,
                                       tol, max_basis, orth_length, cap, iters.ctypes.data_as(C.POINTER(C.c_long)),
                                       _p(amax), C.byref(steps), C.byref(status), C.byref(bus), C.byref(mx),
                                       C.byref(tot), snapshot_every, _p(snaps), _p(snap_t), scap, C.byref(nsn)))
    n_ok = steps.value if status.value == 0 else steps.value - 1
    res = IntegrationResult(u, steps.value, "completed" if status.value == 0 else "blew_up", bus.value, mx.value,
                            tot.value, iters[:n_ok].copy(), amax[:n_ok].copy(), 0.0)
    res.snapshots = [(float(snap_t[k]), snaps[k].copy()) for k in range(min(nsn.value, scap))]
    return res


def phi_combination_dense(A, b_list, dt, tol=1e-12, max_basis=128, orth_length=128):
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    b = np.ascontiguousarray(np.stack(b_list), dtype=np.float64)
    out = np.empty(n)
    iters, subs, est = C.c_long(), C.c_int(), C.c_double()
    _check(lib().oracle_phi_dense_op(n, _p(A), len(b_list) - 1, _p(b), dt, tol, max_basis,
                                     orth_length, _p(out), C.byref(iters), C.byref(subs),
                                     C.byref(est)))
    return out, iters.value, subs.value


def expm(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    out = np.empty_like(A)
    lib().oracle_expm(A.shape[0], _p(A), _p(out))
    return out


def phi_dense_family(p, A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    out = np.empty((p + 1, n, n))
    lib().oracle_phi_dense_family(p, n, _p(A), _p(out))
    return out


def phi_scalar(i, tau):
    return lib().oracle_phi_scalar(i, tau)


def lgl(order):
    n = order + 1
    x, w, D = np.empty(n), np.empty(n), np.empty((n, n))
    _check(lib().oracle_lgl(order, _p(x), _p(w), _p(D)))
    return x, w, D


def gauss(npts):
    x, w = np.empty(npts), np.empty(npts)
    _check(lib().oracle_gauss(npts, _p(x), _p(w)))
    return x, w


def krylov_build(A, seed, m, orth_length):
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    seed = np.ascontiguousarray(seed, dtype=np.float64)
    basis = np.zeros((n, m + 1))
    hess = np.zeros((m + 1, m))
    mo, inv, sn = C.c_int(), C.c_int(), C.c_double()
    _check(lib().oracle_krylov_build(n, _p(A), _p(seed), m, orth_length, _p(basis), _p(hess),
                                     C.byref(mo), C.byref(inv), C.byref(sn)))
    k = mo.value
    cols = k + (0 if inv.value else 1)
    return basis[:, :cols], hess[:k + 1, :k], k, bool(inv.value), sn.value


def euler_pointwise(what, qm, qp=None, n=(1.0, 0.0), gamma=1.4):
    qm = np.ascontiguousarray(qm, dtype=np.float64)
    qp = np.ascontiguousarray(qp if qp is not None else qm, dtype=np.float64)
    out = np.zeros(16)
    _check(lib().oracle_euler_pointwise(what, _p(qm), _p(qp), n[0], n[1], gamma, _p(out)))
    return out


def burgers_flux(kind, um, up, jump, sigma=0.0, h=1.0):
    return lib().oracle_burgers_flux(1 if kind in ("ef", "entropy") else 0, um, up, jump, sigma, h)


def vortex(x, y, t, params, gamma=1.4):
    p = np.ascontiguousarray(params, dtype=np.float64)
    out = np.empty(4)
    lib().oracle_vortex(x, y, t, _p(p), gamma, _p(out))
    return out


def initial_condition(cfg: int, nx: int, order: int, seed: int, noise: float = 1e-6) -> np.ndarray:
    comps = {1: 1, 2: 1, 3: 1, 4: 4, 5: 5}[cfg]
    npe = {1: order + 1, 2: order + 1, 3: (order + 1) ** 2, 4: (order + 1) ** 2,
           5: (order + 1) ** 3}[cfg]
    ne = {1: nx, 2: nx, 3: nx * nx, 4: nx * nx, 5: nx ** 3}[cfg]
    out = np.empty(ne * npe * comps)
    _check(lib().oracle_ic(cfg, nx, order, seed, noise, _p(out)))
    return out


def splitmix_normals(seed, count):
    out = np.empty(count)
    lib().oracle_splitmix_normal(seed, count, _p(out))
    return out


def burgers_diag(problem: Problem, ref, u):
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    q = np.empty(problem.dim)
    vals = [C.c_double() for _ in range(4)]
    _check(lib().oracle_burgers_diag(problem.h, _p(ref), _p(u), _p(q),
                                     *[C.byref(v) for v in vals]))
    return q, tuple(v.value for v in vals)


def burgers_inner(problem: Problem, a, b):
    """<a, b> in the Burgers operator's mass inner product (checker for device residuals)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = C.c_double()
    _check(lib().oracle_burgers_inner(problem.h, _p(a), _p(b), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- harness helpers (checker side)
def harness_burgers(problem, ne, k, flux="", sigma=0.0, sigma_adaptive=False, over_integrate=-1, kappa=-1.0):
    """u0, weak source and effective config of make_problem (proj/src/harness.cpp:48-142)."""
    n = ne * (k + 1)
    u0, src, cfg = np.empty(n), np.empty(n), np.empty(5)
    rc = lib().oracle_harness_burgers(problem.encode(), ne, k, flux.encode(), sigma, int(sigma_adaptive),
                                      over_integrate, kappa, _p(u0), _p(src), _p(cfg))
    if rc:
        raise ValueError("harness problem")
    return u0, src, {"kappa": cfg[0], "flux": "ef" if cfg[1] else "lf", "sigma": cfg[2],
                     "sigma_adaptive": bool(cfg[3]), "over_integrate": bool(cfg[4])}


def mms_source(x, kappa):
    """burgers-mms forcing (proj/src/harness.cpp:97-104)."""
    return lib().oracle_mms_source(float(x), float(kappa))


def l2_error_exact(problem, ne, k, u, t, comp=0):
    u = np.ascontiguousarray(u, dtype=np.float64)
    return lib().oracle_l2_error_exact(problem.encode(), ne, k, _p(u), t, comp)


def harness_u0(problem, ne, k):
    """u0 of make_problem (proj/src/harness.cpp:48-142)."""
    n = lib().oracle_harness_u0(problem.encode(), ne, k, None)
    if n < 0:
        raise ValueError("harness problem")
    out = np.empty(n)
    lib().oracle_harness_u0(problem.encode(), ne, k, _p(out))
    return out


def rk4_reference(problem, ne, k, flux, over_integrate, dt, t_final):
    out = np.empty(ne * (k + 1))
    _check(lib().oracle_rk4_reference(problem.encode(), ne, k, flux.encode(), over_integrate, dt, t_final, _p(out)))
    return out


def l2_error_discrete(problem, ne, k, u, ref_ne, ref_k, uref):
    u = np.ascontiguousarray(u, dtype=np.float64)
    uref = np.ascontiguousarray(uref, dtype=np.float64)
    return lib().oracle_l2_error_discrete(problem.encode(), ne, k, _p(u), ref_ne, ref_k, _p(uref))
