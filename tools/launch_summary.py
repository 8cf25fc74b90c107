"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][-70:]
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "usecond":
            v *= 1e3
        elif d["Metric Unit"] == "msecond":
            v *= 1e6
        agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% |")
