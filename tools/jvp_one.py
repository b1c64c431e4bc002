import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
w = configs.scaled(configs.ALL["C4"], 1024, steps=1)
u0 = torch.tensor(w.initial_condition(), device="cuda:0")
ctx = pkg.Context(0, orth="dcgs2")
op = pkg.Operator(ctx, w.spec())
op.linearize(u0)
print(ctx.bench_apply(op, 10, 2, reps=5))
