"""Per-kernel means of an ncu --csv metrics capture of the branch kernels
(scripts/gpu_ncu.sh, last command): DRAM bytes and executed DADD / DMUL /
DFMA per launch, plus the per-iteration branch-phase FP64 total — the
roofline cross-check bench.py reads (profiles/r02_ncu_traffic.jsonl).
usage: ncu_traffic.py <fp64_counts.csv> > profiles/r02_ncu_traffic.jsonl"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr, body = rows[0], rows[1:]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
TO_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
per = collections.defaultdict(dict)  # (kernel, launch id) -> metric -> value
for r in body:
    name = r[ix["Kernel Name"]]
    k = next((n for n in ("lane_kernel", "tile_kernel", "solo_kernel") if n in name), None)
    if k is None:
        continue
    name_m, v = r[ix["Metric Name"]], float(r[ix["Metric Value"]].replace(",", ""))
    if name_m == "gpu__time_duration.sum":
        v *= TO_US.get(r[ix["Metric Unit"]], 1.0)  # microseconds
    per[(k, int(r[ix["ID"]]))][name_m] = v

M = {"us": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
     "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
     "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"}
tot = collections.Counter()
for k in ("lane_kernel", "tile_kernel", "solo_kernel"):
    ls = [v for (kk, _), v in sorted(per.items()) if kk == k]
    if not ls:
        continue
    mean = {a: sum(l.get(m, 0.0) for l in ls) / len(ls) for a, m in M.items()}
    us = mean["us"]
    print(json.dumps({"kernel": k, "launches": len(ls), "mean_us": us,
                      "dram_read_bytes": mean["rd"], "dram_write_bytes": mean["wr"],
                      "dram_bytes": mean["rd"] + mean["wr"], "dadd": mean["dadd"],
                      "dmul": mean["dmul"], "dfma": mean["dfma"]}))
    for a in ("dadd", "dmul", "dfma"):
        tot[a] += mean[a]
    tot["us"] += us
flops = tot["dadd"] + tot["dmul"] + 2 * tot["dfma"]
print(json.dumps({"kernel": "branch_phase_fp64",
                  "note": "lane+tile+solo per ADMM iteration, mean over inner iterations 1-12 of the "
                          "70k-shaped cold start (ncu, serialized launches); flops = DADD + DMUL + "
                          "2 DFMA (DFMA only inside IEEE div/sqrt sequences)",
                  "dadd": tot["dadd"], "dmul": tot["dmul"], "dfma": tot["dfma"], "flops": flops,
                  "sum_mean_us": tot["us"],
                  "executed_tflops_under_ncu": flops / (tot["us"] * 1e-6) / 1e12 if tot["us"] else None}))
