"""compute-sanitizer target: a few inner iterations of the 2868-shaped grid
with lane_budget = 1 and tile_budget = 1, so nearly every branch is handed
lane -> tile -> solo (every hand-off and shared-slot path runs), then the
device extraction of a short solve.  usage: sanitize_target.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
net = ga.Network(synth.ensure_case("case2868rte", "/tmp/gridadmm_cases"))
cfg = ga.Config(rho_pq=50.0, rho_va=5e3, lane_budget=1, tile_budget=1)
s = ga.Session(net, cfg)
rec, _ = s.iterate(iters)
print("iterations", len(rec), rec[-1, :3])
st, rep = ga.solve(net, ga.Config(rho_pq=50.0, rho_va=5e3, max_outer=1, max_inner=2))
print("solve", st, rep.metrics())
