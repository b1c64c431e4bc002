"""Regenerates the golden fixtures of tests/golden/ (run from the repo root:
`python tests/golden/make_golden.py`).

* acceptance_digits.json — the digits the reference printed in its own acceptance
  run (proj/test_output.txt:18-28), the pins of tests/test_oracle_pins.py and
  tests/test_gpu_acceptance.py.
* *.npz — end states of the oracle (the CPU restatement of the reference, itself
  pinned to those digits) on small seeded problems of the BASELINE configs, with
  per-step cumulative Krylov iterations: the device is checked against these on the
  GPU box (tests/test_gpu_golden.py) and the oracle must keep reproducing them bit
  for bit (tests/test_golden.py).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

DIGITS = {
    "source": "proj/test_output.txt:18-28",
    "criterion_2": {"k2_errors": ["2.455e-06", "3.051e-07", "3.807e-08", "4.755e-09"],
                    "k2_orders": ["3.008", "3.003", "3.001"], "k4_orders": ["5.003", "5.001", "5.000"]},
    "criterion_3": {"orders": ["3.077", "3.019", "3.005"]},
    "criterion_4": {"epi2_orders": ["1.974", "2.044", "2.037"], "epi2_err_dt0.01": "4.942e-06",
                    "exprb32_orders": ["2.641", "2.881", "3.001"]},
    "criterion_5": {"cr_d": "161.0", "epi2_max_ratio": "1.0000", "rk2_blow_up_step": 18},
    "criterion_8": {"rho_orders": {"1": "1.725", "2": "2.709", "3": "3.781"}, "k2_err": "1.486e-05"},
    "criterion_9": {"ode_orders": ["1.09", "2.18", "3.06", "4.16"], "burgers_orders": ["1.04", "2.04", "2.88", "3.70"]},
    "criterion_10": {"errors": ["8.303e-03", "3.847e-03", "1.866e-03"]},
}

# (file, config, nx, steps, integrator)
CASES = [
    ("c1s_nx64_epi2_5steps", "C1s", 64, 5, "epi2"),
    ("c1s_nx64_exprb42_3steps", "C1s", 64, 3, "exprb42"),
    ("c3_nx6_epi2_2steps", "C3", 6, 2, "epi2"),
    ("c4_nx8_epi2_2steps", "C4", 8, 2, "epi2"),
    ("c5_nx3_epi2_1step", "C5", 3, 1, "epi2"),
]


def generate(case):
    from paper_2011_01316_b200 import configs
    from tests.gpu_util import oracle_problem
    name, cfg, nx, steps, integ = case
    w = configs.scaled(configs.ALL[cfg], nx, steps=steps)
    u0 = w.initial_condition()
    dt = w.time_step(u0) if w.dt is None else w.dt
    r = oracle_problem(w.spec()).integrate(integ, u0, dt, steps * dt, tol=w.tol, max_basis=w.max_basis,
                                           orth_length=w.max_basis)
    return dict(u0=u0, u=r.u, dt=np.float64(dt), iters=np.asarray(r.iters_per_step, dtype=np.int64),
                status=np.array(r.status))


if __name__ == "__main__":
    with open(os.path.join(HERE, "acceptance_digits.json"), "w") as f:
        json.dump(DIGITS, f, indent=1)
    for case in CASES:
        np.savez_compressed(os.path.join(HERE, case[0] + ".npz"), **generate(case))
        print("wrote", case[0])
