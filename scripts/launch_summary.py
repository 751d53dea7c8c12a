"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = collections.defaultdict(dict)
names = {}
for r in data:
    d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki].split("(")[0][:44]
agg = collections.defaultdict(list)
for k, v in d.items():
    agg[names[k]].append(v)
for n, l in agg.items():
    t = sum(x["gpu__time_duration.sum"] for x in l) / len(l)
    rb = sum(x.get("dram__bytes_read.sum", 0) for x in l) / len(l)
    wb = sum(x.get("dram__bytes_write.sum", 0) for x in l) / len(l)
    print(f"{n:46s} n={len(l):3d} mean={t / 1e3:9.1f}us dram_read={rb / 1e6:8.2f}MB dram_write={wb / 1e6:8.2f}MB")
