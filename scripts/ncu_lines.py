"""Join ncu per-SASS-instruction samples with nvdisasm line info.
usage: ncu_lines.py <report.ncu-rep> <object.o> <kernel-substring> [callee-substring ...]
The kernel's own function and any listed callees (noinline device functions)
are concatenated in that order and aligned with ncu's SASS rows."""
import csv, io, re, subprocess, sys, collections, os, tempfile
rep, obj = sys.argv[1], sys.argv[2]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
# per function: list of (offset, line-tag)
funcs = collections.OrderedDict(); cur = None; tag = "?"
for ln in sass.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m: cur = m.group(1); funcs[cur] = []; continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m: tag = f"{os.path.basename(m.group(1))}:{m.group(2)}"; continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m and cur: funcs[cur].append((int(m.group(1), 16), tag, m.group(2).strip()))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; data = []
for r in rows:
    if r and r[0] == "Address": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"): data.append(dict(zip(hdr, r)))
print("ncu rows", len(data), "funcs", {k[-40:]: len(v) for k, v in funcs.items()})
# align: ncu lists kernel function then callees in address order; match by sass text sequence
allins = []
for sub in sys.argv[3:]:
    for k, v in funcs.items():
        if sub in k:
            allins += [(k, off, tag, txt) for off, tag, txt in v]
agg = collections.Counter(); inst = collections.Counter(); tot = 0
REASONS = ["stall_no_inst", "stall_wait", "stall_long_sb", "stall_short_sb", "stall_branch_resolving", "stall_selected"]
byr = collections.defaultdict(collections.Counter); rtot = collections.Counter()
n = min(len(allins), len(data))
mismatch = 0
for i in range(n):
    k, off, tag, txt = allins[i]
    d = data[i]
    op_ncu = d["Source"].split()[0] if d["Source"].split() else ""
    op_dis = txt.split()[0] if txt.split() else ""
    if op_ncu.lstrip("@!P0123456789T") and op_ncu != op_dis and not op_dis.startswith("@"): mismatch += 1
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    agg[tag] += s; inst[tag] += float(d["Instructions Executed"] or 0); tot += s
    for r in REASONS:
        v = float(d.get(r) or 0)
        byr[tag][r] += v; rtot[r] += v
print("mismatched opcodes", mismatch, "of", n)
print("stall totals:", {r[6:]: int(v) for r, v in rtot.items()})
for tag, s in agg.most_common(45):
    rs = " ".join(f"{r[6:]}={int(byr[tag][r])}" for r in REASONS if byr[tag][r] > 0.05 * s)
    print(f"{tag:24s} samples {s:8.0f} ({100*s/tot:5.1f}%)  inst {inst[tag]:12.0f}  {rs}")
