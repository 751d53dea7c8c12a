"""GPU time-to-converge of a synthetic shape through gridadmm_solve (preset
penalties, default tolerances), best of R runs after one warm-up solve;
for A/B of build variants via GRIDADMM_LIB.
usage: converge_time.py [shape] [preset] [repeats]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else shape
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))


def config(**kw):
    if ":" in preset:  # explicit "rho_pq:rho_va"
        rpq, rva = (float(v) for v in preset.split(":"))
        return ga.Config(rho_pq=rpq, rho_va=rva, **kw)
    return ga.Config(preset, **kw)


ga.solve(net, config(max_outer=1, max_inner=3))
times = []
for _ in range(reps):
    t0 = time.perf_counter()
    st, rep = ga.solve(net, config())
    times.append(time.perf_counter() - t0)
m = rep.metrics()
print(json.dumps({"lib": os.path.basename(ga.LIB_PATH), "shape": shape, "preset": preset,
                  "status": ga.STATUS[st], "times_s": times, "best_s": min(times),
                  "inner": m["inner_iterations"], "objective_hex": float(m["objective"]).hex(),
                  "c_inf": m["c_inf"]}))
