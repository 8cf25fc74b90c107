"""Opcode mix and stall reasons of one kernel from an ncu report's SASS
source page (read here, no GPU):
  python tools/sass_mix.py report.ncu-rep units [top]
prints warp-instructions per unit (e.g. per prompt) by opcode and the
stall-reason totals."""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
h = None
ops, stalls = collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    src = d["Source"].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    f = lambda k: float(d.get(k, "0").replace(",", "") or 0)
    ops[op.split(".")[0]] += f("Instructions Executed")
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            stalls[k] += f(k)
n = sum(ops.values())
print(f"total warp-instructions {n:.4g} ({n / units:.1f} per unit)")
for k, v in ops.most_common(top):
    print(f"  {k:12s} {100 * v / n:6.2f}%  {v / units:8.1f}")
s = sum(stalls.values())
print("stall samples by reason:")
for k, v in stalls.most_common(12):
    print(f"  {k:24s} {100 * v / s:6.2f}%")
