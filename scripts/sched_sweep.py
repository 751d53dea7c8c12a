"""Branch-schedule knobs (results never depend on them) vs the time to
converge of a synthetic shape: lane_budget / lane_cap / tile_budget /
tail_num combinations, best of 2 solves each.
usage: sched_sweep.py <shape> <preset> '<json list of {key: value}>'"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape, preset, combos = sys.argv[1], sys.argv[2], json.loads(sys.argv[3])


def config(**kw):
    if ":" in preset:  # explicit "rho_pq:rho_va"
        rpq, rva = (float(v) for v in preset.split(":"))
        return ga.Config(rho_pq=rpq, rho_va=rva, **kw)
    return ga.Config(preset, **kw)


net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
ga.solve(net, config(max_outer=1, max_inner=3))
for kw in combos:
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        st, rep = ga.solve(net, config(**kw))
        times.append(time.perf_counter() - t0)
    m = rep.metrics()
    print(json.dumps({"cfg": kw, "best_s": min(times), "inner": m["inner_iterations"],
                      "objective_hex": float(m["objective"]).hex()}), flush=True)
