"""Per-source-line stall samples / shared-memory wavefronts of an ncu report captured with
--import-source on (kernels compiled with -lineinfo): python tools/ncu_lines.py REPORT [top]."""
import csv
import io
import subprocess
import sys


def num(v):
    try:
        return int(v)
    except ValueError:
        return 0


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
per = {}
f = "?"
si = wi = ii = ei = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        si = r.index("# Samples")
        wi = r.index("L1 Wavefronts Shared")
        ii = r.index("L1 Wavefronts Shared Ideal")
        ei = r.index("Instructions Executed")
        continue
    if r[0] not in ("", "Function Name") and si is not None:
        key = (f, num(r[0]), r[1].strip()[:85])
        a = per.setdefault(key, [0, 0, 0, 0])
        a[0] += num(r[si])
        a[1] += num(r[wi])
        a[2] += num(r[ii])
        a[3] += num(r[ei])
tot = sum(v[0] for v in per.values()) or 1
print("samples", tot, "shared wavefronts", sum(v[1] for v in per.values()), "instructions", sum(v[3] for v in per.values()))
for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:20]}:{k[1]:5d} {v[0]:6d} {100 * v[0] / tot:5.1f}%  wf {v[1] / 1e6:6.2f}M (ideal {v[2] / 1e6:6.2f}M) "
          f"inst {v[3] / 1e6:6.2f}M  {k[2]}")
