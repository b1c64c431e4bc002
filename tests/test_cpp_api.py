"""The header-only C++ mirror (include/expdg_b200.hpp) compiles against the
C ABI and links the in-tree library; host setup runs without a GPU."""
import os
import subprocess

import pytest

import paper_2011_01316_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build_example():
    lib = pkg.build()
    libdir = os.path.dirname(lib)
    out = os.path.join(libdir, "integrate_vortex")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "integrate_vortex.cpp"), "-L", libdir, "-lexpdg_b200",
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    return out


def test_cpp_example_builds_and_runs_host_setup():
    exe = _build_example()
    r = subprocess.run([exe, "--host-only"], capture_output=True, text=True, check=True)
    assert "lgl nodes[1]" in r.stdout


@pytest.mark.gpu
def test_cpp_example_integrates_on_device():
    exe = _build_example()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "status=completed steps=3" in r.stdout
