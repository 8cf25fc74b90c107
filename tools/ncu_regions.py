"""Per-region totals of an ncu source page (read here, no GPU): warp-stall
samples and executed warp-instructions summed over line ranges of one file.
  python tools/ncu_regions.py report.ncu-rep file.cu name:lo-hi [name:lo-hi ...]
Lines outside every range are reported per line (top 15) under 'other'."""
import collections
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0])
cur, hs = None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hs = r
        continue
    if not hs or len(r) != len(hs) or not r[0]:
        continue

    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    a = agg[(cur, int(r[0]))]
    a[0] += f(r[4])
    a[1] += f(r[7])
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
reg = collections.OrderedDict((n, [0.0, 0.0]) for n, _, _ in ranges)
other = {}
for (fl, ln), v in agg.items():
    hit = None
    if fl == fname:
        for n, lo, hi in ranges:
            if lo <= ln <= hi:
                hit = n
                break
    if hit:
        reg[hit][0] += v[0]
        reg[hit][1] += v[1]
    else:
        other[(fl, ln)] = v
print(f"total: {ts:.0f} stall samples, {ti:.4g} warp-instructions")
print("| region | stall % | inst % |\n|---|---|---|")
for n, v in reg.items():
    print(f"| {n} | {100 * v[0] / ts:.1f} | {100 * v[1] / ti:.1f} |")
os_, oi = sum(v[0] for v in other.values()), sum(v[1] for v in other.values())
print(f"| other | {100 * os_ / ts:.1f} | {100 * oi / ti:.1f} |")
for k, v in sorted(other.items(), key=lambda x: -x[1][1])[:15]:
    print(f"|   {k[0]}:{k[1]} | {100 * v[0] / ts:.1f} | {100 * v[1] / ti:.1f} |")
