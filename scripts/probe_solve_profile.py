"""Probe: full cold-start solve with the per-iteration kernel profile
(GRIDADMM_PROFILE) and host phase trace; summarises where the time goes.
usage: probe_solve_profile.py <shape> <rho_pq> <rho_va> [max_inner] [max_outer] [out.csv]"""
import os
import sys
import time

shape = sys.argv[1]
rpq, rva = float(sys.argv[2]), float(sys.argv[3])
max_inner = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
max_outer = int(sys.argv[5]) if len(sys.argv) > 5 else 20
out = sys.argv[6] if len(sys.argv) > 6 else f"/tmp/prof_{shape}.csv"
if os.path.exists(out):
    os.remove(out)
os.environ["GRIDADMM_PROFILE"] = out
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
cfg = ga.Config(rho_pq=rpq, rho_va=rva, max_inner=max_inner, max_outer=max_outer)
t = time.perf_counter()
st, rep = ga.solve(net, cfg)
wall = time.perf_counter() - t
m = rep.metrics()
print(f"{shape} rho=({rpq:g},{rva:g}) {ga.STATUS[st]} inner={m['inner_iterations']:.0f} "
      f"outer={m['outer_iterations']:.0f} c_inf={m['c_inf']:.3g} obj={m['objective']:.8g} wall={wall:.2f}s")
d = np.genfromtxt(out, delimiter=",", names=True)
tot = d["gen_ms"] + d["lane_ms"] + d["tile_ms"] + d["bus_zy_ms"]
print(f"device ms total {tot.sum():.0f}: gen {d['gen_ms'].sum():.0f} lane {d['lane_ms'].sum():.0f} "
      f"tile {d['tile_ms'].sum():.0f} bus {d['bus_zy_ms'].sum():.0f}; host/other {wall * 1e3 - tot.sum():.0f}")
q = np.percentile(tot, [50, 90, 99, 100])
print("per-iteration ms p50/90/99/max", np.round(q, 3))
n = len(d)
for a in range(0, n, max(1, n // 20)):
    sl = slice(a, min(n, a + max(1, n // 20)))
    print(f"  it {a:6d}: mean {tot[sl].mean():7.3f} ms lane {d['lane_ms'][sl].mean():7.3f} "
          f"tile {d['tile_ms'][sl].mean():7.3f} ovf6 {d['ovf6'][sl].mean():7.0f} ovf4 {d['ovf4'][sl].mean():7.0f} "
          f"beta {d['beta'][sl].max():.3g}")
