"""Fused JVP + DCGS2-dots sweep vs the separate passes, per Krylov column j.

python tools/fusedbench.py [nx] [j,j,...] [C3|C4|C5] : for each j, ms of the JVP alone (EXPDG_E2_DOTS=0 /
EXPDG_E3_DOTS=0), the DCGS2 dots pass, the fused sweep, and (C4) the fused sweep with the dot arithmetic
skipped (EXPDG_E2_DBG=1).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_01316_b200 as pkg  # noqa: E402
from paper_2011_01316_b200 import configs  # noqa: E402


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    js = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 4, 10, 20, 30, 40]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "C4"
    w = configs.scaled(configs.ALL[cfg], nx, steps=1)
    dv = {"C4": "EXPDG_E2_DOTS", "C5": "EXPDG_E3_DOTS", "C3": "EXPDG_B2_DOTS"}[cfg]
    u0 = torch.tensor(w.initial_condition(), device="cuda:0")
    ctx = pkg.Context(0, orth="dcgs2")
    ops = {}
    for name, env in (("jvp", {dv: "0"}), ("fused", {dv: "1"}), ("fused_nofma", {dv: "1", "EXPDG_E2_DBG": "1"}),
                      *((("fused_dbg", {dv: "1", "EXPDG_E2_DBG": os.environ["FB_DBG"]}),) if "FB_DBG" in os.environ else ())):
        for k in ("EXPDG_E2_DOTS", "EXPDG_E3_DOTS", "EXPDG_B2_DOTS", "EXPDG_E2_DBG"):
            os.environ.pop(k, None)
        os.environ.update(env)
        op = pkg.Operator(ctx, w.spec())
        op.linearize(u0)
        ops[name] = op
    n = ops["jvp"].dim
    for j in js:
        r = {"j": j, "n": n}
        r["jvp_ms"] = ctx.bench_apply(ops["jvp"], j, 0)
        r["dots_ms"] = ctx.bench_apply(ops["jvp"], j, 1)
        r["fused_ms"] = ctx.bench_apply(ops["fused"], j, 0)
        r["fused_nofma_ms"] = ctx.bench_apply(ops["fused_nofma"], j, 0)
        if "fused_dbg" in ops:
            r["fused_dbg_ms"] = ctx.bench_apply(ops["fused_dbg"], j, 0)
        gb_f = 8.0 * n * (j + 4) / 1e9
        r["fused_GBps"] = gb_f / r["fused_ms"] * 1e3
        r["separate_ms"] = r["jvp_ms"] + r["dots_ms"]
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
