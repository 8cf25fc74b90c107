"""Per-source-line instruction counts of an ncu report, grouped into line
ranges (phases). Usage: python tools/ncu_phases.py rep.ncu-rep file.cu n_units a-b:name ..."""
import collections
import csv
import io
import subprocess
import sys

rep, fname, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
ranges = []
for a in sys.argv[4:]:
    r, name = a.split(":")
    lo, hi = r.split("-")
    ranges.append((int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = line = None
agg = collections.Counter()
tot = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:
        line = (cur, int(r[0]))
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        n = int(r[7] or 0)
        agg[line] += n
        tot += n
g = collections.Counter()
for (f, l), n in agg.items():
    if f != fname:
        g["other:" + f] += n
        continue
    for lo, hi, name in ranges:
        if lo <= l <= hi:
            g[name] += n
            break
    else:
        g["line%d" % l] += n
print(f"total warp-instructions {tot:.4g}, per unit {tot / units:.1f}")
for k, v in g.most_common(25):
    print(f"{k:40s} {v:12d} {100 * v / tot:5.1f}%  per unit {v / units:8.1f}")
