"""Median duration per kernel of an ncu --csv launch list: python tools/launch_split.py FILE"""
import collections
import csv
import sys

rows = list(csv.DictReader(line for line in open(sys.argv[1]) if line.startswith('"')))
agg = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        agg[r["Kernel Name"][:100]].append(v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    v.sort()
    print(f"{len(v):5d} launches  median {v[len(v) // 2]:10.1f} us  {k}")
