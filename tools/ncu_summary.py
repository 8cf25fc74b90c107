"""Summarise an ncu report (read here, no GPU): speed-of-light, occupancy,
dram bytes, and the top source lines by warp-stall samples / instructions.
Usage: python tools/ncu_summary.py report.ncu-rep [top_n] > profiles/<name>.md"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


details = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = details[0]
kernels = collections.OrderedDict()
for r in details[1:]:
    d = dict(zip(h, r))
    k = (d.get("ID"), d.get("Kernel Name", "")[:90])
    kernels.setdefault(k, []).append(d)
want = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Size", "Grid Size", "Theoretical Occupancy", "Achieved Occupancy",
        "Achieved Active Warps Per SM", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Avg. Active Threads Per Warp", "No Eligible"]
for (kid, name), rows in kernels.items():
    print(f"## kernel {kid}: `{name}`\n")
    print("| metric | value |\n|---|---|")
    seen = set()
    for d in rows:
        m = d["Metric Name"]
        if m in want and m not in seen:
            seen.add(m)
            print(f"| {m} | {d['Metric Value']} {d['Metric Unit']} |")
    print()
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
if raw:
    hh = raw[0]
    for r in raw[2:]:
        d = dict(zip(hh, r))
        rd = d.get("dram__bytes_read.sum", "")
        wr = d.get("dram__bytes_write.sum", "")
        print(f"raw: kernel `{d.get('Kernel Name','')[:60]}` dram__bytes_read.sum={rd} "
              f"({raw[1][hh.index('dram__bytes_read.sum')] if 'dram__bytes_read.sum' in hh else ''}) "
              f"dram__bytes_write.sum={wr}\n")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
cur = None
hs = None
for r in src:
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
    a[2] = r[1].strip()[:100]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"\n### top {top} source lines by warp-stall samples (total {ts:.0f} samples, {ti:.3g} warp-instr)\n")
print("| file:line | stall % | inst % | source |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"| {k[0]}:{k[1]} | {100*v[0]/ts:.1f} | {100*v[1]/ti:.1f} | `{v[2]}` |")
