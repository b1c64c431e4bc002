"""One workload's pipelined-DCGS2 lookahead JVP (stage 2) per launch: python tools/jvp_one.py [C3|C4|C5] [nx]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
base = configs.ALL[cfg]
nx = int(sys.argv[2]) if len(sys.argv) > 2 else base.nx
w = configs.scaled(base, nx, steps=1)
u0 = torch.tensor(w.initial_condition(), device="cuda:0")
ctx = pkg.Context(0, orth="dcgs2")
op = pkg.Operator(ctx, w.spec())
op.linearize(u0)
ms = ctx.bench_apply(op, 10, 2, reps=20)
print(f"{cfg} nx {nx}: {ms * 1e3:.1f} us per launch, {32.0 * w.dofs / ms / 1e6:.0f} GB/s of algorithmic bytes")
