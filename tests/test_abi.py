"""CPU-side checks of the drop-in boundary: the C-ABI library builds for
sm_100a, loads, and exports every symbol include/expdg_b200.h declares."""
import ctypes
import os
import re

import pytest

import paper_2011_01316_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "expdg_b200.h")).read()
    return sorted(set(re.findall(r"\b(expdg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exports():
    assert set(_declared()) == set(pkg.EXPORTS)


def test_library_builds_and_exports_every_symbol():
    path = pkg.build()
    assert os.path.exists(path)
    L = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(L, name), name


def test_sm100a_cubin_present():
    import subprocess
    path = pkg.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_setup_matches_oracle_bit_for_bit():
    import numpy as np
    import oracle
    for k in (1, 3, 4, 7):
        a = pkg.lgl_basis(k)
        b = oracle.lgl(k)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for cfg, nx, order in [(1, 64, 4), (2, 64, 7), (3, 8, 4), (4, 8, 4), (5, 3, 3)]:
        seed = 1234 + cfg
        u_dev_side = pkg.initial_condition(cfg, nx, order, seed, 1e-6)
        u_oracle = oracle.initial_condition(cfg, nx, order, seed, 1e-6)
        assert np.array_equal(u_dev_side, u_oracle), cfg


def test_invalid_arguments_map_to_value_error_without_gpu():
    with pytest.raises(ValueError):
        pkg.lgl_basis(0)
    with pytest.raises(ValueError):
        pkg.initial_condition(9, 4, 4, 1)


def test_tgv_slab_generator_matches_global_state():
    # the per-rank C5 slabs (bench.py --config C5L at N > 1) concatenate to the global state
    import numpy as np
    import paper_2011_01316_b200 as pkg
    from paper_2011_01316_b200 import configs
    full = pkg.initial_condition(5, 6, 3, 0, 0.0)
    parts = [pkg.initial_condition_slab(5, 6, 6, 6, 3, a, b) for a, b in ((0, 1), (1, 4), (4, 6))]
    assert np.array_equal(np.concatenate(parts), full)
    w = configs.scaled(configs.C5L, 4, nz=8)
    assert np.array_equal(np.concatenate([w.initial_condition_slab(0, 3), w.initial_condition_slab(3, 8)]),
                          w.initial_condition())
