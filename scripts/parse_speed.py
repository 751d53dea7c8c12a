"""MATPOWER parse time, product parser (network.cpp, single pass) vs the
reference's (netdata.cpp:124-230), on the same synthetic files through each
library's gridadmm_network_load (host only; median of 5).
usage: parse_speed.py [out.json]"""
import ctypes
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402


def timed(load, free, path, reps=5):
    ts = []
    for _ in range(reps):
        h = ctypes.c_void_p()
        t0 = time.perf_counter()
        assert load(os.fsencode(path), ctypes.byref(h)) == 0
        ts.append(time.perf_counter() - t0)
        free(h)
    return statistics.median(ts)


ref = oracle.ref_capi()
mine = ga.lib()
out = []
for shape in ("case2868rte", "case9241pegase", "case_ACTIVSg25k", "case_ACTIVSg70k"):
    path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
    r = timed(ref.gridadmm_network_load, ref.gridadmm_network_free, path)
    m = timed(mine.gridadmm_network_load, mine.gridadmm_network_free, path)
    out.append({"shape": shape, "bytes": os.path.getsize(path), "reference_s": r, "product_s": m,
                "speedup": r / m})
    print(json.dumps(out[-1]), flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump({"host": os.uname().nodename, "cpus": os.cpu_count(), "runs": out}, f, indent=1)
