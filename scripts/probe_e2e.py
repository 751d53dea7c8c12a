"""Probe: fixed cost of gridadmm_solve on the 70k-shaped grid (engine setup,
upload, cold start, solution download) vs per-iteration cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

p = synth.ensure_case("case_ACTIVSg70k", "/tmp/gridadmm_cases")
net = ga.Network(p)
for n in (1, 1, 5, 50, 200, 200):
    cfg = ga.Config("case_ACTIVSg70k", max_outer=1, max_inner=n)
    t = time.perf_counter()
    st, rep = ga.solve(net, cfg)
    dt = time.perf_counter() - t
    rep.write_convergence("/tmp/e2e_conv.csv")
    el = np.loadtxt("/tmp/e2e_conv.csv", delimiter=",", skiprows=1, ndmin=2)[:, 5]
    print(f"max_inner={n:4d} wall={dt * 1e3:8.1f} ms first_elapsed={el[0] * 1e3:7.1f} ms "
          f"last_elapsed={el[-1] * 1e3:8.1f} ms", flush=True)
