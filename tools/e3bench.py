"""The C5 z-march JVP per launch (the pipelined DCGS2 lookahead application, stage 2, and the
stage-1 sweep with the fused dots at column j): python tools/e3bench.py [nx] [j]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 64
j = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = configs.scaled(configs.C5, nx, steps=1)
u0 = torch.tensor(w.initial_condition(), device="cuda:0")
ctx = pkg.Context(0, orth="dcgs2")
op = pkg.Operator(ctx, w.spec())
op.linearize(u0)
n = w.dofs
st2 = ctx.bench_apply(op, j, 2, reps=20)
st1 = ctx.bench_apply(op, j, 0, reps=20)
print(json.dumps({"n": n, "j": j, "stage2_ms": round(st2, 4), "stage2_GBps": round(32.0 * n / st2 / 1e6, 1),
                  "stage1_dots_ms": round(st1, 4), "stage1_GBps": round(8.0 * n * (4 + j) / st1 / 1e6, 1)}))
