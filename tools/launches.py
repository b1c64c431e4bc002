"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import io
import sys


def summarise(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"]) / 1e6
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} {c:5d} launches {t:10.2f} ms {100 * t / tot:6.2f}%  avg {t / c:8.3f} ms")
    out.append(f"total {tot:.2f} ms over {sum(c for c, _ in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
