"""SASS census of a built object: per kernel, instruction count and the
source lines with the most local-memory (spill) instructions.
usage: sass_census.py <object.o> [kernel-substring]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
cur, tag = None, "?"
spill = collections.defaultdict(collections.Counter)
lines = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for ln in sass.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        tag = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m and cur:
        ops = [o for o in m.group(2).split() if not o.startswith("@")]
        op = ops[0] if ops else ""
        tot[cur] += 1
        lines[cur][tag] += 1
        if op.startswith(("STL", "LDL")):
            spill[cur][(tag, op.split(".")[0])] += 1
for f in tot:
    if sub not in f:
        continue
    print(f"{f[-60:]}: {tot[f]} instructions, {sum(spill[f].values())} local ld/st")
    for (t, o), c in spill[f].most_common(12):
        print(f"    {t:28s} {o} {c}")
    print("    largest lines:", ", ".join(f"{t} {c}" for t, c in lines[f].most_common(10)))
