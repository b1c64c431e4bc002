import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2011_01316_b200 as pkg
from paper_2011_01316_b200 import configs
for cfg, env in (("C4", "EXPDG_E2_RHS_TILE"), ("C5", "EXPDG_E3_RHS_TILE")):
    w = configs.ALL[cfg]
    u0 = torch.tensor(w.initial_condition(), device="cuda:0")
    for v in ("0", "1"):
        os.environ[env] = v
        ctx = pkg.Context(0)
        op = pkg.Operator(ctx, w.spec())
        y = op.full_rhs(u0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the library launches on its own stream: time by wall clock around synchronised calls
        t = time.perf_counter()
        for _ in range(10):
            y = op.full_rhs(u0)
        torch.cuda.synchronize()
        print(cfg, "tile" if v == "1" else "strip/march", round((time.perf_counter() - t) * 100, 3), "ms per full_rhs (incl. the output allocation)", flush=True)
