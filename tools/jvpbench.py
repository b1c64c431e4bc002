"""The pipelined DCGS2 lookahead JVP (stage 2) per launch at C4 size: the plain strip kernel as
run (half-width strips, EXPDG_E2_CW2=4), at full width (EXPDG_E2_CW2=8), and without its face
fluxes (EXPDG_E2_DBG=4: wrong results, the time the face phase costs); cw4_fw is the default
(face warps, EXPDG_E2_FW=0 turns them off)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
w = configs.scaled(configs.ALL[cfg], nx, steps=1)
u0 = torch.tensor(w.initial_condition(), device="cuda:0")
ctx = pkg.Context(0, orth="dcgs2")
variants = {"cw4_fw": {"EXPDG_E2_CW2": "4", "EXPDG_E2_FW": "1"},
            "cw4_fw_align": {"EXPDG_E2_CW2": "4", "EXPDG_E2_FW": "1", "EXPDG_E2_ALIGN": "1"}, "cw4": {"EXPDG_E2_CW2": "4", "EXPDG_E2_FW": "0"},
            "cw8": {"EXPDG_E2_CW2": "8"},
            "cw4_nofaces": {"EXPDG_E2_CW2": "4", "EXPDG_E2_DBG": "4", "EXPDG_E2_FW": "0"},
            "cw8_nofaces": {"EXPDG_E2_CW2": "8", "EXPDG_E2_DBG": "4"}}
res = {}
for name, env in variants.items():
    for k in ("EXPDG_E2_CW2", "EXPDG_E2_DBG", "EXPDG_E2_FW", "EXPDG_E2_ALIGN"):
        os.environ.pop(k, None)
    os.environ.update(env)
    op = pkg.Operator(ctx, w.spec())
    op.linearize(u0)
    res[name] = ctx.bench_apply(op, 10, 2, reps=10)
n = w.dofs
print(json.dumps({"n": n, **{k: round(v, 4) for k, v in res.items()},
                  "GBps_cw4": round(32.0 * n / res["cw4"] / 1e6, 1),
                  "GBps_cw4_fw": round(32.0 * n / res["cw4_fw"] / 1e6, 1)}))
