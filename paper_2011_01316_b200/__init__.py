"""paper_2011_01316_b200 — B200-native exponential-DG hot path.

Python mirror of the reference library's operator API (/root/reference/proj,
`expdg`): split-operator factory + linearize (burgers_split_operator /
euler_split_operator), the JVP `apply_linear`, `apply_nonlinear`,
`full_rhs`, `phi_combination`, `step_epi2` and `integrate`, all executed by
the sm_100a CUDA library `_build/libexpdg_b200.so` through its C ABI
(include/expdg_b200.h).  There is no CPU fallback: without the built library
and a CUDA device every call raises.

PyTorch is plumbing only (device memory and streams).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# EXPDG_LIB: another in-tree build of the same library (same-box A/B of kernel variants)
LIB_PATH = os.environ.get("EXPDG_LIB") or os.path.join(_PKG, "_build", "libexpdg_b200.so")

EXPDG_OK, EXPDG_E_INVALID, EXPDG_E_DOMAIN, EXPDG_E_KRYLOV, EXPDG_E_CUDA, EXPDG_E_UNSUPPORTED, EXPDG_E_COMM = range(7)
BURGERS1D, BURGERS2D, EULER2D, EULER3D, DENSE = 1, 2, 3, 4, 5
INTEGRATORS = {"exp_euler": 0, "epi2": 1, "exprb32": 2, "exprb42": 3}


class KrylovError(RuntimeError):
    """proj/include/expdg/phi.hpp:61-66 — carries the last error estimate."""

    def __init__(self, msg, last_estimate=0.0):
        super().__init__(msg)
        self.last_estimate = last_estimate


class DeviceError(RuntimeError):
    pass


class UnsupportedError(ValueError):
    pass


class CommError(DeviceError):
    """A communicator call (NCCL / local group) of the multi-GPU path failed."""


class OpDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("order", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("z0", C.c_double), ("z1", C.c_double), ("periodic", C.c_int), ("kappa", C.c_double),
        ("flux", C.c_int), ("sigma", C.c_double), ("sigma_adaptive", C.c_int),
        ("over_integrate", C.c_int), ("gamma", C.c_double), ("euler_flux", C.c_int),
        ("part_begin", C.c_int), ("part_end", C.c_int),
        ("grade_x", C.POINTER(C.c_double)), ("grade_y", C.POINTER(C.c_double)), ("grade_z", C.POINTER(C.c_double)),
    ]


class KrylovCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_basis", C.c_int), ("orth_length", C.c_int),
                ("initial_basis", C.c_int), ("max_substeps", C.c_int)]


class KrylovStatsC(C.Structure):
    _fields_ = [("iterations", C.c_longlong), ("substeps", C.c_int), ("last_estimate", C.c_double)]


ON_STEP_FN = C.CFUNCTYPE(None, C.c_int, C.c_double, C.c_double, C.c_longlong, C.c_void_p)


class TimeCfg(C.Structure):
    _fields_ = [("integrator", C.c_int), ("dt", C.c_double), ("t_final", C.c_double),
                ("krylov", KrylovCfg), ("use_graph", C.c_int), ("snapshot_every", C.c_int),
                ("snapshot_cap", C.c_int), ("snapshots", C.c_void_p), ("snapshot_times", C.POINTER(C.c_double)),
                ("on_step", ON_STEP_FN), ("on_step_user", C.c_void_p)]


class IntegrationResultC(C.Structure):
    _fields_ = [("t", C.c_double), ("status", C.c_int), ("steps", C.c_int),
                ("krylov_iterations", C.c_longlong), ("blow_up_step", C.c_int), ("max_abs", C.c_double),
                ("snapshots", C.c_int)]


# user LinearAction / SplitProblem callbacks on device vectors (include/expdg_b200.h expdg_user_op_fns)
USER_APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
USER_LINEARIZE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class UserOpFns(C.Structure):
    _fields_ = [("apply_linear", USER_APPLY_FN), ("apply_nonlinear", USER_APPLY_FN),
                ("linearize", USER_LINEARIZE_FN), ("graph_safe", C.c_int)]


# symbols declared in include/expdg_b200.h (checked by tests/test_abi.py)
EXPORTS = [
    "expdg_last_error", "expdg_ctx_create", "expdg_ctx_destroy", "expdg_ctx_stream", "expdg_ctx_synchronize",
    "expdg_op_create", "expdg_dense_op_create", "expdg_op_destroy", "expdg_op_dim", "expdg_op_linearize",
    "expdg_op_apply_linear", "expdg_op_apply_nonlinear", "expdg_op_full_rhs", "expdg_phi_combination",
    "expdg_step_epi2", "expdg_integrate", "expdg_integrate_host", "expdg_lgl_basis",
    "expdg_initial_condition", "expdg_ctx_kernel_launches", "expdg_ctx_last_loop_ms", "expdg_expm",
    "expdg_debug_state", "expdg_debug_hessenberg", "expdg_ctx_traffic", "expdg_bench_ts", "expdg_bench_apply", "expdg_op_set_source",
    "expdg_op_set_source_fn", "expdg_nccl_unique_id", "expdg_ctx_attach_nccl", "expdg_local_group_create",
    "expdg_local_group_destroy", "expdg_ctx_attach_local", "expdg_ctx_comm", "expdg_ctx_set_orthogonalization",
    "expdg_debug_profile", "expdg_debug_expm_profile", "expdg_ctx_set_fused", "expdg_ctx_time_dominant", "expdg_ctx_dominant_stats",
    "expdg_ctx_last_path", "expdg_user_op_create", "expdg_krylov_build", "expdg_initial_condition_slab",
    "expdg_ctx_set_pipelined", "expdg_peer_group_create", "expdg_peer_group_destroy", "expdg_ctx_attach_peer_local",
    "expdg_ctx_peer_export", "expdg_ctx_attach_peer",
]

_lib = None
SOURCE_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)


def build(force: bool = False) -> str:
    from . import _build
    return _build.build(force=force)


def lib():
    """Loads the CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"expdg CUDA library missing: {LIB_PATH} (run paper_2011_01316_b200._build)")
    L = C.CDLL(LIB_PATH)
    vp, dp, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_longlong
    L.expdg_last_error.restype = C.c_char_p
    L.expdg_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.expdg_ctx_destroy.argtypes = [vp]
    L.expdg_ctx_stream.restype = vp
    L.expdg_ctx_stream.argtypes = [vp]
    L.expdg_ctx_synchronize.argtypes = [vp]
    L.expdg_ctx_kernel_launches.restype = i64
    L.expdg_ctx_kernel_launches.argtypes = [vp]
    L.expdg_ctx_last_loop_ms.restype = C.c_double
    L.expdg_ctx_last_loop_ms.argtypes = [vp]
    L.expdg_op_create.argtypes = [vp, C.POINTER(OpDesc), C.POINTER(vp)]
    L.expdg_dense_op_create.argtypes = [vp, C.c_int, dp, C.POINTER(vp)]
    L.expdg_op_destroy.argtypes = [vp]
    L.expdg_op_dim.restype = i64
    L.expdg_op_dim.argtypes = [vp]
    L.expdg_op_linearize.argtypes = [vp, vp]
    L.expdg_op_set_source.argtypes = [vp, vp]
    L.expdg_op_set_source_fn.argtypes = [vp, SOURCE_FN, vp]
    for f in ("expdg_op_apply_linear", "expdg_op_apply_nonlinear", "expdg_op_full_rhs"):
        getattr(L, f).argtypes = [vp, vp, vp, vp]
    L.expdg_phi_combination.argtypes = [vp, vp, C.POINTER(vp), C.c_int, C.c_double, C.POINTER(KrylovCfg), vp,
                                        C.POINTER(KrylovStatsC)]
    L.expdg_step_epi2.argtypes = [vp, vp, vp, C.c_double, C.POINTER(KrylovCfg), C.POINTER(KrylovStatsC)]
    L.expdg_integrate.argtypes = [vp, vp, vp, C.POINTER(TimeCfg), C.POINTER(IntegrationResultC),
                                  C.POINTER(i64), dp, C.c_int]
    L.expdg_integrate_host.argtypes = [vp, vp, dp, C.POINTER(TimeCfg), C.POINTER(IntegrationResultC),
                                       C.POINTER(i64), dp, C.c_int]
    L.expdg_lgl_basis.argtypes = [C.c_int, dp, dp, dp]
    L.expdg_expm.argtypes = [vp, C.c_int, dp, dp]
    L.expdg_debug_state.argtypes = [vp, dp]
    L.expdg_debug_hessenberg.argtypes = [vp, dp]
    L.expdg_ctx_traffic.argtypes = [vp, dp]
    L.expdg_bench_ts.argtypes = [vp, C.c_longlong, C.c_int, C.c_int, C.c_int, dp]
    L.expdg_bench_apply.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, dp]
    L.expdg_initial_condition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, dp]
    L.expdg_initial_condition_slab.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp, C.c_int, C.c_int,
                                               dp]
    L.expdg_nccl_unique_id.argtypes = [C.c_char_p]
    L.expdg_ctx_attach_nccl.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
    L.expdg_local_group_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.expdg_local_group_destroy.argtypes = [vp]
    L.expdg_ctx_attach_local.argtypes = [vp, vp, C.c_int]
    L.expdg_ctx_comm.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.expdg_ctx_set_orthogonalization.argtypes = [vp, C.c_int]
    L.expdg_debug_profile.argtypes = [vp, C.POINTER(C.c_longlong)]
    L.expdg_debug_expm_profile.argtypes = [vp, C.POINTER(C.c_longlong)]
    L.expdg_ctx_set_fused.argtypes = [vp, C.c_int]
    L.expdg_ctx_set_pipelined.argtypes = [vp, C.c_int]
    L.expdg_peer_group_create.argtypes = [C.c_int, C.c_longlong, C.POINTER(vp)]
    L.expdg_peer_group_destroy.argtypes = [vp]
    L.expdg_ctx_attach_peer_local.argtypes = [vp, vp, C.c_int]
    L.expdg_ctx_peer_export.argtypes = [vp, C.c_int, C.c_longlong, C.c_char_p]
    L.expdg_ctx_attach_peer.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
    L.expdg_ctx_time_dominant.argtypes = [vp, C.c_int]
    L.expdg_ctx_dominant_stats.argtypes = [vp, dp]
    L.expdg_ctx_last_path.argtypes = [vp, C.POINTER(C.c_int)]
    L.expdg_user_op_create.argtypes = [vp, C.c_longlong, C.POINTER(UserOpFns), vp, C.POINTER(vp)]
    L.expdg_krylov_build.argtypes = [vp, vp, vp, C.c_int, C.c_int, vp, dp, dp, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
    _lib = L
    return L


import threading as _threading

_user_exc = _threading.local()  # the Python exception a user-operator callback raised last


def _check(rc, stats: Optional[KrylovStatsC] = None):
    if rc == EXPDG_OK:
        return
    msg = lib().expdg_last_error().decode()
    exc = getattr(_user_exc, "e", None)
    if exc is not None:
        _user_exc.e = None
        msg = f"{msg} ({type(exc).__name__}: {exc})"
    if rc == EXPDG_E_INVALID:
        raise ValueError(msg)
    if rc == EXPDG_E_DOMAIN:
        raise ArithmeticError(msg)
    if rc == EXPDG_E_KRYLOV:
        raise KrylovError(msg, stats.last_estimate if stats is not None else 0.0)
    if rc == EXPDG_E_UNSUPPORTED:
        raise UnsupportedError(msg)
    if rc == EXPDG_E_COMM:
        raise CommError(msg)
    raise DeviceError(msg)


def _dptr(t) -> int:
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return t.data_ptr()


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------- setup helpers
def lgl_basis(order: int):
    """proj/src/basis.cpp:35-85 (host setup of the device constants)."""
    n = order + 1
    x, w, D = np.empty(n), np.empty(n), np.empty((n, n))
    _check(lib().expdg_lgl_basis(order, _np_ptr(x), _np_ptr(w), _np_ptr(D)))
    return x, w, D


def initial_condition(config: int, nx: int, order: int, seed: int, noise: float = 1e-6) -> np.ndarray:
    """Seeded synthetic input of BASELINE.json config C<config>."""
    if config not in (1, 2, 3, 4, 5):
        raise ValueError("initial_condition: config must be 1..5")
    comps = {1: 1, 2: 1, 3: 1, 4: 4, 5: 5}[config]
    npe = {1: order + 1, 2: order + 1, 3: (order + 1) ** 2, 4: (order + 1) ** 2, 5: (order + 1) ** 3}[config]
    ne = {1: nx, 2: nx, 3: nx * nx, 4: nx * nx, 5: nx ** 3}[config]
    out = np.empty(ne * npe * comps)
    _check(lib().expdg_initial_condition(config, nx, order, seed, noise, _np_ptr(out)))
    return out


def initial_condition_slab(config: int, nx: int, ny: int, nz: int, order: int, layer_begin: int, layer_end: int,
                           box=(0.0, 2 * math.pi, 0.0, 2 * math.pi, 0.0, 2 * math.pi)) -> np.ndarray:
    """Config 5's Taylor-Green state, z-planes [layer_begin, layer_end) of an nx x ny x nz mesh
    (the owned slab of a z-partitioned rank)."""
    npe = (order + 1) ** 3
    out = np.empty((layer_end - layer_begin) * nx * ny * npe * 5)
    b6 = np.ascontiguousarray(box, dtype=np.float64)
    _check(lib().expdg_initial_condition_slab(config, nx, ny, nz, order, _np_ptr(b6), layer_begin, layer_end,
                                              _np_ptr(out)))
    return out


# ---------------------------------------------------------------- context / operators
class Context:
    def __init__(self, device: int = 0, orth: Optional[str] = None, fused: Optional[bool] = None,
                 pipelined: Optional[bool] = None):
        """orth: None (auto: DCGS2 from 2^18 DOF up), "dcgs2" or "cgs2" for fully orthogonalised phi calls;
        fused: None / True runs small 1D Burgers phi calls as one single-CTA kernel, False never;
        pipelined: None / True streams the basis once per DCGS2 column (lookahead application), False
        runs the two-pass DCGS2."""
        import torch
        torch.cuda.init()
        self.device = device
        h = C.c_void_p()
        _check(lib().expdg_ctx_create(device, C.byref(h)))
        self.h = h
        if orth is not None:
            if orth not in ("cgs2", "dcgs2"):
                raise ValueError("orth must be 'cgs2' or 'dcgs2'")
            _check(lib().expdg_ctx_set_orthogonalization(self.h, 1 if orth == "dcgs2" else 0))
        if fused is not None:
            _check(lib().expdg_ctx_set_fused(self.h, 1 if fused else 0))
        if pipelined is not None:
            _check(lib().expdg_ctx_set_pipelined(self.h, 1 if pipelined else 0))

    def close(self):
        if getattr(self, "h", None):
            lib().expdg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return lib().expdg_ctx_kernel_launches(self.h)

    @property
    def last_loop_ms(self) -> float:
        return lib().expdg_ctx_last_loop_ms(self.h)

    def expm(self, a: np.ndarray) -> np.ndarray:
        """The device controller's expm (proj/src/phi.cpp:40 restated, Higham 2005)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty_like(a)
        _check(lib().expdg_expm(self.h, a.shape[0], _np_ptr(a), _np_ptr(out)))
        return out

    def debug_state(self) -> dict:
        v = np.zeros(16)
        _check(lib().expdg_debug_state(self.h, _np_ptr(v)))
        keys = ["mc", "h", "t", "beta", "avnorm", "last_estimate", "substeps", "iterations", "breakdown",
                "status", "mmax", "grow_cap", "full_orth", "cycles", "pre_norm", "m"]
        return dict(zip(keys, v.tolist()))

    def traffic(self) -> dict:
        """Canonical algorithmic bytes of the last call's realised trajectory."""
        v = np.zeros(4)
        _check(lib().expdg_ctx_traffic(self.h, _np_ptr(v)))
        return {"alg_bytes": v[0], "columns": int(v[1]), "avnorms": int(v[2]), "combines": int(v[3])}

    def bench_apply(self, op: "Operator", j: int, mode: int = 0, reps: int = 5) -> float:
        """avg ms of one phi-cycle operator application at column j (mode 0, with the DCGS2
        dots where the operator kernel takes them) or of the DCGS2 dots pass (mode 1)."""
        ms = C.c_double()
        _check(lib().expdg_bench_apply(self.h, op.h, j, mode, reps, C.byref(ms)))
        return ms.value

    def bench_ts(self, n: int, k: int, mode: int, reps: int = 5) -> float:
        """avg ms of one CGS2 streaming pass (0 dots, 1 update+dots, 2 update+norm, 3 combine)."""
        ms = C.c_double()
        _check(lib().expdg_bench_ts(self.h, n, k, mode, reps, C.byref(ms)))
        return ms.value

    def time_dominant(self, enable=True):
        """CUDA events around every DCGS2 update pass (enable True / 1) or every phi-cycle
        operator application (2) of the next host-stepped runs; False / 0: off."""
        _check(lib().expdg_ctx_time_dominant(self.h, int(enable)))

    def dominant_stats(self) -> dict:
        v = np.zeros(3)
        _check(lib().expdg_ctx_dominant_stats(self.h, _np_ptr(v)))
        return {"ms": v[0], "bytes": v[1], "launches": int(v[2])}

    def last_path(self) -> dict:
        """Engine path of the last phi / integrate call."""
        v = (C.c_int * 4)()
        _check(lib().expdg_ctx_last_path(self.h, v))
        return {"dcgs2": bool(v[0]), "pipelined": v[0] == 2, "fused_dots": bool(v[1]), "graph": bool(v[2]),
                "fused_engine": bool(v[3])}

    def debug_profile(self) -> dict:
        """Fused small-problem engine: SM cycles per phase of the last run."""
        v = (C.c_longlong * 8)()
        _check(lib().expdg_debug_profile(self.h, v))
        return dict(zip(["apply", "dots", "update", "combine", "control", "expm", "expm_calls"], list(v)[:7]))

    def debug_expm_profile(self) -> dict:
        """SM cycles of the controller's expm sub-phases, summed over its calls."""
        v = (C.c_longlong * 8)()
        _check(lib().expdg_debug_expm_profile(self.h, v))
        return dict(zip(["norm_scale", "pade", "lu", "backsub", "squarings", "calls", "squarings_taken"], list(v)[:7]))

    def debug_hessenberg(self) -> np.ndarray:
        h = np.zeros((129, 128))
        _check(lib().expdg_debug_hessenberg(self.h, _np_ptr(h)))
        return h

    def synchronize(self):
        _check(lib().expdg_ctx_synchronize(self.h))

    # ---- multi-GPU slab partition
    def attach_nccl(self, unique_id: bytes, rank: int, size: int):
        """Collective over the `size` ranks (ncclCommInitRank); unique_id from nccl_unique_id()."""
        _check(lib().expdg_ctx_attach_nccl(self.h, bytes(unique_id), rank, size))
        return self

    def attach_local(self, group: "LocalGroup", rank: int):
        """Rank `rank` of a host-staged group driven by threads of this process."""
        self._group = group  # keep the group alive as long as the context
        _check(lib().expdg_ctx_attach_local(self.h, group.h, rank))
        return self

    def attach_peer_local(self, group: "PeerGroup", rank: int):
        """Rank `rank` of a device-resident peer-memory group of threads of this process."""
        self._group = group
        _check(lib().expdg_ctx_attach_peer_local(self.h, group.h, rank))
        return self

    def peer_export(self, size: int, halo_doubles: int) -> bytes:
        """One process per GPU: allocate this rank's peer region; returns its 64-byte CUDA IPC handle."""
        buf = C.create_string_buffer(64)
        _check(lib().expdg_ctx_peer_export(self.h, size, halo_doubles, buf))
        return buf.raw

    def attach_peer(self, handles: Sequence[bytes], rank: int, size: int):
        """Map the peers' regions (all ranks' handles in rank order) and attach the communicator."""
        blob = b"".join(bytes(h) for h in handles)
        _check(lib().expdg_ctx_attach_peer(self.h, blob, rank, size))
        return self

    @property
    def comm(self) -> tuple:
        r, n = C.c_int(), C.c_int()
        _check(lib().expdg_ctx_comm(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().expdg_nccl_unique_id(buf))
    return buf.raw


class PeerGroup:
    """Device-resident peer-memory communicator group for several ranks in one process (one device)."""

    def __init__(self, size: int, halo_doubles: int = 1 << 20):
        h = C.c_void_p()
        _check(lib().expdg_peer_group_create(size, halo_doubles, C.byref(h)))
        self.h = h
        self.size = size

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().expdg_peer_group_destroy(self.h)
                self.h = None
        except Exception:
            pass


class LocalGroup:
    """Host-staged communicator group for several ranks in one process (single-GPU tests)."""

    def __init__(self, size: int):
        h = C.c_void_p()
        _check(lib().expdg_local_group_create(size, C.byref(h)))
        self.h = h
        self.size = size

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().expdg_local_group_destroy(self.h)
                self.h = None
        except Exception:
            pass


@dataclass
class OperatorSpec:
    kind: str  # burgers1d | burgers2d | euler2d | euler3d
    order: int
    nx: int
    ny: int = 1
    nz: int = 1
    box: tuple = (0.0, 1.0, 0.0, 1.0, 0.0, 1.0)
    periodic: bool = True
    kappa: float = 0.03
    flux: str = "lf"
    sigma: float = 0.0
    sigma_adaptive: bool = False
    over_integrate: bool = False
    gamma: float = 1.4
    euler_flux: str = "lf"
    part: tuple = (0, 0)  # owned element rows [begin, end) of a slab-partitioned 2D Euler mesh
    # grading lists of build_quad_mesh (proj/src/mesh.cpp:96-120): nx+1 / ny+1 (/ nz+1) breakpoints
    grade_x: Optional[Sequence[float]] = None
    grade_y: Optional[Sequence[float]] = None
    grade_z: Optional[Sequence[float]] = None

    def desc(self) -> OpDesc:
        d = OpDesc()
        d.kind = {"burgers1d": BURGERS1D, "burgers2d": BURGERS2D, "euler2d": EULER2D, "euler3d": EULER3D}[self.kind]
        d.order, d.nx, d.ny, d.nz = self.order, self.nx, self.ny, self.nz
        d.x0, d.x1, d.y0, d.y1, d.z0, d.z1 = self.box
        d.periodic = int(self.periodic)
        d.kappa, d.flux, d.sigma = self.kappa, (1 if self.flux in ("ef", "entropy") else 0), self.sigma
        d.sigma_adaptive, d.over_integrate = int(self.sigma_adaptive), int(self.over_integrate)
        d.gamma, d.euler_flux = self.gamma, (0 if self.euler_flux == "roe" else 1)
        d.part_begin, d.part_end = self.part
        # the library copies the lists at creation; keep them alive until then
        d._grades = [None if g is None else np.ascontiguousarray(g, dtype=np.float64)
                     for g in (self.grade_x, self.grade_y, self.grade_z)]
        d.grade_x, d.grade_y, d.grade_z = [None if g is None else _np_ptr(g) for g in d._grades]
        return d

    @property
    def components(self) -> int:
        return {"burgers1d": 1, "burgers2d": 1, "euler2d": 4, "euler3d": 5}[self.kind]


class Operator:
    """A DG operator on the device; `linearize(ref)` freezes u~ like the
    reference split-operator factories (proj/src/burgers.cpp:309-320)."""

    def __init__(self, ctx: Context, spec: Optional[OperatorSpec] = None, dense=None):
        self.ctx = ctx
        self.spec = spec
        h = C.c_void_p()
        if dense is not None:
            a = np.ascontiguousarray(dense, dtype=np.float64)
            _check(lib().expdg_dense_op_create(ctx.h, a.shape[0], _np_ptr(a), C.byref(h)))
        else:
            d = spec.desc()
            _check(lib().expdg_op_create(ctx.h, C.byref(d), C.byref(h)))
        self.h = h
        self.dim = lib().expdg_op_dim(h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().expdg_op_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def linearize(self, ref):
        import torch
        torch.cuda.current_stream().synchronize()
        _check(lib().expdg_op_linearize(self.h, _dptr(ref)))
        return self

    def set_source(self, weak_source):
        """BurgersConfig::source as its weak load vector (proj/src/burgers.cpp:80-92)."""
        import torch
        torch.cuda.current_stream().synchronize()
        _check(lib().expdg_op_set_source(self.h, _dptr(weak_source)))
        return self

    def set_source_function(self, source):
        """BurgersConfig::source given as a callable s(x) (proj/include/expdg/burgers.hpp:22);
        the library builds the weak load on its own quadrature (proj/src/burgers.cpp:80-92)."""
        cb = SOURCE_FN(lambda x, _user: float(source(x)))
        _check(lib().expdg_op_set_source_fn(self.h, cb, None))
        return self

    def _apply(self, fn, x, out=None):
        import torch
        out = torch.empty_like(x) if out is None else out
        stream = torch.cuda.current_stream().cuda_stream
        _check(getattr(lib(), fn)(self.h, _dptr(x), _dptr(out), C.c_void_p(stream)))
        return out

    def apply_linear(self, x, out=None):
        """SplitOperator::linear — the JVP (proj/src/burgers.cpp:146-180, euler.cpp:299-341)."""
        return self._apply("expdg_op_apply_linear", x, out)

    def apply_nonlinear(self, x, out=None):
        return self._apply("expdg_op_apply_nonlinear", x, out)

    def full_rhs(self, x, out=None):
        return self._apply("expdg_op_full_rhs", x, out)


class _DeviceVector:
    """A device pointer of n doubles seen by torch (no copy): __cuda_array_interface__."""

    def __init__(self, ptr, n, readonly=False):
        # torch accepts only writable views; `readonly` documents intent (the library never reads them back)
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


def _status_of(exc) -> int:
    if isinstance(exc, ArithmeticError):
        return EXPDG_E_DOMAIN
    if isinstance(exc, ValueError):
        return EXPDG_E_INVALID
    return EXPDG_E_CUDA


class SplitProblem:
    """A user SplitProblem (proj/include/expdg/integrators.hpp:48-52) on device vectors:
    `linearize(ref) -> (linear, nonlinear)` like the reference's factory, where `ref` is a
    read-only CUDA tensor and `linear(x) -> y` / `nonlinear(x) -> y` act on CUDA tensors
    (`nonlinear` may be None: N = 0).  A plain LinearAction is `SplitProblem(n, linear=f)`.
    Raise ArithmeticError for the reference's std::domain_error (integrate then reports
    blew_up) and ValueError for std::invalid_argument.  The callables run on the engine's
    stream (it is torch's current stream inside them).  graph_safe=True lets the library
    record them once into its CUDA graphs: the actions then take `(x, out)` and write into
    `out`, enqueueing only allocation-free stream work (e.g. torch ops with `out=` buffers)."""

    def __init__(self, dim: int, linearize=None, linear=None, nonlinear=None, graph_safe: bool = False):
        if linearize is None and linear is None:
            raise ValueError("SplitProblem: need linearize(ref) -> (linear, nonlinear) or a fixed linear action")
        self.dim, self.graph_safe = int(dim), graph_safe
        self._linearize, self._linear, self._nonlinear = linearize, linear, nonlinear


class UserOperator:
    """Operator of a user SplitProblem on the device engine (expdg_user_op_create)."""

    def __init__(self, ctx: Context, problem: SplitProblem):
        import torch
        self.ctx, self.problem, self.dim = ctx, problem, problem.dim
        n = problem.dim
        self._L, self._N = problem._linear, problem._nonlinear

        def run(stream, fn):
            try:
                with torch.cuda.stream(torch.cuda.ExternalStream(stream or 0, device=f"cuda:{ctx.device}")):
                    fn()
                return EXPDG_OK
            except Exception as e:  # noqa: BLE001 — mapped to the reference's exception types
                _user_exc.e = e
                return _status_of(e)

        def vec(p, ro=False):
            return torch.as_tensor(_DeviceVector(p, n, ro), device=f"cuda:{ctx.device}")

        def apply(which):
            def cb(x, y, stream, _user):
                def go():
                    f = self._L if which == 0 else self._N
                    out = vec(y)
                    if f is None:
                        out.zero_()
                    elif problem.graph_safe:
                        f(vec(x, True), out)  # graph-safe actions write into `out`
                    else:
                        out.copy_(f(vec(x, True)))
                return run(stream, go)
            return cb

        def lin_cb(ref, stream, _user):
            def go():
                r = problem._linearize(vec(ref, True))
                self._L, self._N = (r if isinstance(r, tuple) else (r, None))
            return run(stream, go)

        self._cbs = (USER_APPLY_FN(apply(0)), USER_APPLY_FN(apply(1)),
                     USER_LINEARIZE_FN(lin_cb) if problem._linearize is not None else USER_LINEARIZE_FN())
        f = UserOpFns()
        f.apply_linear, f.apply_nonlinear, f.linearize = self._cbs
        f.graph_safe = 1 if problem.graph_safe else 0
        h = C.c_void_p()
        _check(lib().expdg_user_op_create(ctx.h, n, C.byref(f), None, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().expdg_op_destroy(self.h)
                self.h = None
        except Exception:
            pass

    linearize = None  # set below (shared with Operator)


for _m in ("linearize", "_apply", "apply_linear", "apply_nonlinear", "full_rhs"):
    setattr(UserOperator, _m, getattr(Operator, _m))


def _kcfg(tol, max_basis, orth_length, initial_basis=0, max_substeps=0) -> KrylovCfg:
    k = KrylovCfg()
    k.tol, k.max_basis, k.orth_length = tol, max_basis, orth_length
    k.initial_basis, k.max_substeps = initial_basis, max_substeps
    return k


@dataclass
class KrylovStats:
    iterations: int = 0
    substeps: int = 0
    last_estimate: float = 0.0


def phi_combination(ctx: Context, op: Operator, b: Sequence, dt: float, tol: float = 1e-12,
                    max_basis: int = 128, orth_length: int = 128, initial_basis: int = 16,
                    max_substeps: int = 40, out=None):
    """proj/src/phi.cpp:133-260: sum_i dt^i phi_i(dt L) b_i; entries of b may be None (zero)."""
    import torch
    if len(b) == 0:
        raise ValueError("phi_combination: empty b list")
    torch.cuda.current_stream().synchronize()
    ptrs = (C.c_void_p * len(b))(*[C.c_void_p(_dptr(x) if x is not None else 0) for x in b])
    if out is None:
        out = torch.empty(op.dim, dtype=torch.float64, device=f"cuda:{ctx.device}")
    st = KrylovStatsC()
    cfg = _kcfg(tol, max_basis, orth_length, initial_basis, max_substeps)
    rc = lib().expdg_phi_combination(ctx.h, op.h, ptrs, len(b) - 1, dt, C.byref(cfg), C.c_void_p(_dptr(out)),
                                     C.byref(st))
    _check(rc, st)
    return out, KrylovStats(st.iterations, st.substeps, st.last_estimate)


def step_epi2(ctx: Context, op: Operator, u, dt: float, tol=1e-12, max_basis=128, orth_length=128):
    """proj/src/integrators.cpp:76-83 (u updated in place and returned)."""
    import torch
    torch.cuda.current_stream().synchronize()
    st = KrylovStatsC()
    cfg = _kcfg(tol, max_basis, orth_length)
    _check(lib().expdg_step_epi2(ctx.h, op.h, C.c_void_p(_dptr(u)), dt, C.byref(cfg), C.byref(st)), st)
    return u, KrylovStats(st.iterations, st.substeps, st.last_estimate)


@dataclass
class IntegrationResult:
    """proj/include/expdg/integrators.hpp:66-74."""
    u: object
    t: float
    status: str
    steps: int
    krylov_iterations: int
    blow_up_step: int
    max_abs: float
    iters_per_step: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    amax_per_step: np.ndarray = field(default_factory=lambda: np.zeros(0))
    loop_ms: float = 0.0
    snapshots: list = field(default_factory=list)  # [(t, u)] every snapshot_every steps


def integrate(ctx: Context, op, u0, integrator: str, dt: float, t_final: float, tol=1e-12,
              max_basis=128, orth_length=128, use_graph: bool = True, snapshot_every: int = 0,
              on_step=None) -> IntegrationResult:
    """proj/src/integrators.cpp:140-201 on the device.  `u0` may be a CUDA
    tensor (updated in place) or a host numpy array (copied in/out inside the call).
    snapshot_every / on_step(step, t, max_abs, krylov_iterations): TimeLoopConfig
    (proj/include/expdg/integrators.hpp:58-63); on_step runs as each step completes."""
    import torch
    cfg = TimeCfg()
    cfg.integrator = INTEGRATORS[integrator]
    cfg.dt, cfg.t_final = dt, t_final
    cfg.krylov = _kcfg(tol, max_basis, orth_length)
    cfg.use_graph = int(use_graph)
    cap = int(math.ceil(t_final / dt + 1e-9)) + 2
    iters = np.zeros(cap, dtype=np.int64)
    amax = np.zeros(cap)
    host = isinstance(u0, np.ndarray)
    n = op.dim
    scap = cap // snapshot_every if snapshot_every > 0 else 0
    snap_t = np.zeros(max(scap, 1))
    snaps = None
    if scap:
        snaps = np.zeros((scap, n)) if host else torch.empty((scap, n), dtype=torch.float64, device=u0.device)
        cfg.snapshot_every, cfg.snapshot_cap = snapshot_every, scap
        cfg.snapshots = snaps.ctypes.data if host else snaps.data_ptr()
        cfg.snapshot_times = _np_ptr(snap_t)
    cb = None
    if on_step is not None:
        cb = ON_STEP_FN(lambda s_, t_, a_, it_, _u: on_step(s_, t_, a_, it_))
        cfg.on_step = cb
    res = IntegrationResultC()
    if host:
        u = np.ascontiguousarray(u0, dtype=np.float64)
        _check(lib().expdg_integrate_host(ctx.h, op.h, _np_ptr(u), C.byref(cfg), C.byref(res),
                                          iters.ctypes.data_as(C.POINTER(C.c_longlong)), _np_ptr(amax), cap))
    else:
        u = u0
        torch.cuda.current_stream().synchronize()
        _check(lib().expdg_integrate(ctx.h, op.h, C.c_void_p(_dptr(u)), C.byref(cfg), C.byref(res),
                                     iters.ctypes.data_as(C.POINTER(C.c_longlong)), _np_ptr(amax), cap))
    n_ok = res.steps if res.status == 0 else res.steps - 1
    out = IntegrationResult(u, res.t, "completed" if res.status == 0 else "blew_up", res.steps,
                            res.krylov_iterations, res.blow_up_step, res.max_abs, iters[:n_ok].copy(),
                            amax[:n_ok].copy(), ctx.last_loop_ms)
    out.snapshots = [(float(snap_t[k]), snaps[k]) for k in range(min(res.snapshots, scap))]
    return out


@dataclass
class KrylovFactorization:
    """proj/include/expdg/phi.hpp:30-36."""
    basis: object        # CUDA tensor n x (m + 1) (n x m on an invariant subspace)
    hessenberg: np.ndarray  # (m + 1) x m
    seed_norm: float
    m: int
    invariant_subspace: bool


def krylov_build(ctx: Context, op, seed, m: int, orth_length: int) -> KrylovFactorization:
    """proj/src/phi.cpp:115-130 on the device engine: Arnoldi (orth_length >= m) or incomplete
    orthogonalisation of span{seed, L seed, ...}."""
    import torch
    torch.cuda.current_stream().synchronize()
    n = op.dim
    basis = torch.zeros((m + 1, n), dtype=torch.float64, device=f"cuda:{ctx.device}")  # column c = row c
    h = np.zeros((m + 1) * m)
    sn, mo, inv = C.c_double(), C.c_int(), C.c_int()
    _check(lib().expdg_krylov_build(ctx.h, op.h, C.c_void_p(_dptr(seed)), m, orth_length,
                                    C.c_void_p(basis.data_ptr()), _np_ptr(h), C.byref(sn), C.byref(mo),
                                    C.byref(inv)))
    k = mo.value
    cols = k + (0 if inv.value else 1)
    return KrylovFactorization(basis[:cols].T, h[:(k + 1) * k].reshape(k + 1, k).copy(), sn.value, k,
                               bool(inv.value))


from . import configs  # noqa: E402,F401
