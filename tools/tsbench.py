"""Sweep the CGS2 streaming passes: GB/s per (mode, k) under env-selected tuning."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_01316_b200 as pkg

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 104857601
ctx = pkg.Context(0)
res = {}
for k in (5, 20, 40):
    for mode in (0, 1, 2, 3):
        ms = ctx.bench_ts(n, k, mode, 3)
        streams = {0: k + 1, 1: k + 2, 2: k + 2, 3: k + 1}[mode]
        gbs = streams * 8.0 * n / (ms * 1e-3) / 1e9
        res[f"m{mode}k{k}"] = round(gbs)
print(json.dumps({"tuning": {k: os.environ.get(k) for k in ("EXPDG_TS_BUDGET", "EXPDG_TS_STAGES", "EXPDG_TS_MIN_T", "EXPDG_LD_ODD")}, "gbs": res}))
