"""Per-iteration device time of a full cold-start solve (GRIDADMM_PROFILE
csv: gen / lane / tile+solo / bus ms per inner iteration) against the wall
clock of gridadmm_solve: how much of time-to-converge is kernels, and which.
usage: probe_solve_profile.py <shape> <preset> [out.json]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

shape, preset = sys.argv[1], sys.argv[2]


def config(**kw):
    if ":" in preset:  # explicit "rho_pq:rho_va"
        rpq, rva = (float(v) for v in preset.split(":"))
        return ga.Config(rho_pq=rpq, rho_va=rva, **kw)
    return ga.Config(preset, **kw)

prof = os.path.join(tempfile.mkdtemp(), "prof.csv")
os.environ["GRIDADMM_PROFILE"] = prof
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
ga.solve(net, config(max_outer=1, max_inner=2))
open(prof, "w").close()
t0 = time.perf_counter()
st, rep = ga.solve(net, config())
wall = time.perf_counter() - t0
rows = np.genfromtxt(prof, delimiter=",", names=True)
m = rep.metrics()
n = len(rows)
dev = {k: float(np.sum(rows[k])) * 1e-3 for k in ("gen_ms", "lane_ms", "tile_ms", "bus_zy_ms")}
dev_total = sum(dev.values())  # the critical path: the side-stream bus launch overlaps tile_ms
if "bus_side_ms" in rows.dtype.names:
    dev["bus_side_ms_overlapped"] = float(np.sum(rows["bus_side_ms"])) * 1e-3
deciles = []
for q in range(10):
    part = rows[q * n // 10:(q + 1) * n // 10]
    deciles.append({k: float(np.mean(part[k])) for k in ("lane_ms", "tile_ms", "bus_zy_ms")
                    + (("bus_side_ms",) if "bus_side_ms" in rows.dtype.names else ())})
out = {"shape": shape, "preset": preset, "status": ga.STATUS[st], "wall_s": wall,
       "inner_iterations": int(m["inner_iterations"]), "c_inf": m["c_inf"],
       "device_s": dev, "device_total_s": dev_total, "host_gap_s": wall - dev_total,
       "host_gap_us_per_iteration": (wall - dev_total) / max(n, 1) * 1e6,
       "mean_ms_by_decile": deciles}
print(json.dumps(out))
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        json.dump(out, f, indent=1)
