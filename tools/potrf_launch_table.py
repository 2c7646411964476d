"""Summarise an ncu launch list of tools/potrf_once.py: per kernel kind, launches and total us."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows:
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name[:60]
    us = float(r[vi].replace(",", "")) / 1e3
    agg[name][0] += 1
    agg[name][1] += us
    tot += us
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:9.1f} us  {n:4d} launches  {k}")
print(f"{tot:9.1f} us total")
