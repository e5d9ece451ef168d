"""Median duration per kernel from an ncu --metrics gpu__time_duration.sum
--csv launch list: python tools/launch_summary.py LIST.csv [...]"""
import collections
import csv
import statistics
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    ix = {h: i for i, h in enumerate(rows[0])}
    d = collections.defaultdict(list)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        d[name].append(v)
    print(f)
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:40s} n={len(v):5d} median {statistics.median(v):9.2f} us")
