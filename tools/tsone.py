"""One tall-skinny pass (mode, k) at C4 size, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_01316_b200 as pkg

mode, k = int(sys.argv[1]), int(sys.argv[2])
n = int(float(sys.argv[3])) if len(sys.argv) > 3 else 104857601
ctx = pkg.Context(0)
ms = ctx.bench_ts(n, k, mode, 2)
streams = {0: k + 1, 1: k + 2, 2: k + 2, 3: k + 1}[mode]
print(f"mode {mode} k {k}: {ms:.3f} ms, {streams * 8.0 * n / (ms * 1e-3) / 1e9:.0f} GB/s")
