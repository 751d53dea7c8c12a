"""Per-region profile of a branch kernel from an ncu --set full capture: warp
stall samples, warp-level and thread-level instructions executed (their
ratio = active threads per warp) by TRON section, attributing inlined code to
the innermost enclosing section via nvdisasm's inline chains.
usage: ncu_regions.py <report.ncu-rep> <object.o> <kernel-substring>"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, sub = sys.argv[1], sys.argv[2], sys.argv[3]
REGIONS = [  # (file, first line, last line, name): tron.cuh / branch_problem.cuh sections
    ("tron.cuh", 92, 93, "div/sqrt (out of line)"),
    ("tron.cuh", 208, 266, "cauchy search (serial)"),
    ("tron.cuh", 474, 545, "cauchy search (tile)"),
    ("tron.cuh", 270, 370, "subspace CG + Cholesky"),
    ("tron.cuh", 426, 452, "line search (serial)"),
    ("tron.cuh", 547, 575, "line search (tile)"),
    ("tron.cuh", 399, 410, "tron_begin"),
    ("tron.cuh", 578, 665, "tron_step rest / finish"),
    ("branch_problem.cuh", 1, 10000, "branch f / g / H evaluation"),
    ("ga_sincos.h", 1, 10000, "sincos"),
    ("branch.cu", 1, 10000, "schedule / AL / slots"),
]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                      text=True).stdout
funcs = collections.OrderedDict()
cur, chain, pending = None, [], []
for ln in sass.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        f0 = (os.path.basename(m.group(1)), int(m.group(2)))
        if not pending:
            pending = [f0]
        if m.group(3):
            pending.append((os.path.basename(m.group(3)), int(m.group(4))))
        chain = pending
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m and cur:
        pending = []
        funcs[cur].append(list(chain))


def region(ch):
    for f, l in ch:  # innermost first
        for rf, a, b, name in REGIONS:
            if f == rf and a <= l <= b:
                return name
    return "other"


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
        data.append(dict(zip(hdr, r)))
chains = []
for k, v in funcs.items():
    if sub in k:
        chains += v
n = min(len(chains), len(data))
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for i in range(n):
    d = data[i]
    a = agg[region(chains[i])]
    a[0] += float(d["Warp Stall Sampling (All Samples)"] or 0)
    a[1] += float(d["Instructions Executed"] or 0)
    a[2] += float(d["Thread Instructions Executed"] or 0)
ts = sum(v[0] for v in agg.values()) or 1.0
ti = sum(v[1] for v in agg.values()) or 1.0
print(f"{'region':32s} {'samples':>8s} {'%':>6s} {'warp inst':>12s} {'%':>6s} {'threads/warp':>12s}")
for name, (s, wi, th) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{name:32s} {s:8.0f} {100 * s / ts:6.1f} {wi:12.0f} {100 * wi / ti:6.1f} "
          f"{(th / wi if wi else 0):12.1f}")
print(f"{'total':32s} {ts:8.0f} {'':6s} {ti:12.0f} {'':6s} "
      f"{sum(v[2] for v in agg.values()) / ti:12.1f}")
