"""Reference-solution files and experiment CSV in the reference harness formats.

The reference caches its fine-grid reference solutions as text files
("expdg-reference-v1": a key/value header then one "%.17g" value per line,
proj/src/harness.cpp:240-300) and writes experiment tables as CSV
(proj/src/harness.cpp:481-502).  These readers/writers let device results be
cross-validated against files the reference harness produced, and let the
device write files the reference can load.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence

import numpy as np

MAGIC = "expdg-reference-v1"


@dataclass
class ReferenceSpec:
    """proj/include/expdg/harness.hpp:105-117 (same defaults)."""
    problem: str
    flux: str = "lf"
    sigma: float = 0.0
    sigma_adaptive: bool = False
    over_integrate: bool = False
    kappa: float = 0.03
    integrator: str = "rk4"
    k: int = 8
    ne: int = 40
    dt: float = 1e-5
    t_final: float = 1.0

    def components(self) -> int:
        return 4 if self.problem == "euler-vortex" else 1

    def size(self) -> int:
        """State length make_problem builds for this spec (proj/src/harness.cpp:48-142)."""
        if self.problem == "euler-vortex":
            return self.ne * (self.k + 1) ** 2 * 4
        return self.ne * (self.k + 1)


def format_double(v: float) -> str:
    """proj/src/harness.cpp:40-44 ("%.17g")."""
    return "%.17g" % v


def _g(v: float) -> str:
    # std::ostream << double with the default precision 6 (the file-name fields)
    return "%g" % v


def reference_filename(spec: ReferenceSpec) -> str:
    """proj/src/harness.cpp:240-252."""
    name = f"{spec.problem}_{spec.flux}"
    if spec.sigma_adaptive:
        name += "_sadapt"
    elif spec.sigma != 0.0:
        name += f"_s{_g(spec.sigma)}"
    if spec.over_integrate:
        name += "_oi"
    name += (f"_kap{_g(spec.kappa)}_{spec.integrator}_k{spec.k}_ne{spec.ne}_dt{_g(spec.dt)}"
             f"_t{_g(spec.t_final)}.ref")
    return name


def _header(spec: ReferenceSpec, size: int, components: int) -> str:
    # proj/src/harness.cpp:256-272
    return "".join([
        f"{MAGIC}\n", f"problem {spec.problem}\n", f"flux {spec.flux}\n", f"sigma {format_double(spec.sigma)}\n",
        f"sigma_adaptive {1 if spec.sigma_adaptive else 0}\n", f"over_integrate {1 if spec.over_integrate else 0}\n",
        f"kappa {format_double(spec.kappa)}\n", f"integrator {spec.integrator}\n", f"k {spec.k}\n",
        f"ne {spec.ne}\n", f"dt {format_double(spec.dt)}\n", f"t_final {format_double(spec.t_final)}\n",
        f"components {components}\n", f"size {size}\n"])


def save_reference(path: str, spec: ReferenceSpec, values: Sequence[float], components: Optional[int] = None):
    """proj/src/harness.cpp:290-300: written to path.tmp, then renamed (atomic)."""
    values = np.asarray(values, dtype=np.float64).ravel()
    comps = spec.components() if components is None else components
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write(_header(spec, values.size, comps))
        f.write("".join(format_double(float(v)) + "\n" for v in values))
    os.replace(tmp, path)


def load_reference(path: str, expected: ReferenceSpec) -> np.ndarray:
    """proj/src/harness.cpp:302-353: validates every metadata field against `expected`
    (RuntimeError on a mismatch, a truncated file or a size mismatch)."""
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != MAGIC:
        raise RuntimeError(f"reference file format mismatch: {path}")
    hdr, i, size, comps = {}, 1, 0, 0
    while i < len(lines):
        parts = lines[i].split()
        i += 1
        key, value = (parts + ["", ""])[:2]
        hdr[key] = value
        if key == "size":
            size = int(value)
            break
        if key == "components":
            comps = int(value)

    def mismatch(what):
        raise RuntimeError(f"reference metadata mismatch ({what}) in {path}")

    if hdr.get("problem") != expected.problem:
        mismatch("problem")
    if hdr.get("flux") != expected.flux:
        mismatch("flux")
    if float(hdr.get("sigma", "nan")) != expected.sigma:
        mismatch("sigma")
    if int(hdr.get("sigma_adaptive", -1)) != (1 if expected.sigma_adaptive else 0):
        mismatch("sigma_adaptive")
    if int(hdr.get("over_integrate", -1)) != (1 if expected.over_integrate else 0):
        mismatch("over_integrate")
    if float(hdr.get("kappa", "nan")) != expected.kappa:
        mismatch("kappa")
    if hdr.get("integrator") != expected.integrator:
        mismatch("integrator")
    if int(hdr.get("k", -1)) != expected.k:
        mismatch("k")
    if int(hdr.get("ne", -1)) != expected.ne:
        mismatch("ne")
    if float(hdr.get("dt", "nan")) != expected.dt:
        mismatch("dt")
    if float(hdr.get("t_final", "nan")) != expected.t_final:
        mismatch("t_final")
    if size != expected.size() or comps != expected.components():
        raise RuntimeError(f"reference size mismatch in {path}")
    body = lines[i:i + size]
    if len(body) < size or (size and body[-1] == ""):
        raise RuntimeError(f"truncated reference file {path}")
    return np.array([float(v) for v in body], dtype=np.float64)


@dataclass
class ExperimentRow:
    """One row of ExperimentResult (proj/include/expdg/harness.hpp): mesh scale, per-component
    errors and orders (NaN = empty), Courant numbers, Krylov iterations, wall clock, status."""
    scale: float
    error: List[float]
    order: List[float]
    cr_a: float
    cr_d: float
    krylov_iters: int
    wallclock_s: float
    status: str


def experiment_csv(rows: Iterable[ExperimentRow], comp_names: Sequence[str]) -> str:
    """proj/src/harness.cpp:481-495."""
    out = ["scale" + "".join(f",error_{c}" for c in comp_names) + "".join(f",order_{c}" for c in comp_names)
           + ",cr_a,cr_d,krylov_iters,wallclock_s,status\n"]
    for r in rows:
        cells = [format_double(r.scale)]
        cells += [format_double(e) if math.isfinite(e) else "" for e in r.error]
        cells += [format_double(o) if math.isfinite(o) else "" for o in r.order]
        cells += [format_double(r.cr_a), format_double(r.cr_d), str(r.krylov_iters), format_double(r.wallclock_s),
                  r.status]
        out.append(",".join(cells) + "\n")
    return "".join(out)
