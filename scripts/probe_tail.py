"""Probe (stats build, GRIDADMM_LIB=.../libgridadmm_stats.so): per-branch
executed trust-region steps of the lane and tile phases, per ADMM iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
ex = net.export()
limited = ex["branch"][:, 5] > 0
s = ga.Session(net, ga.Config("case_ACTIVSg70k"))
for it in range(n_it):
    ms, rec = s.timed_steps(1, 0)
    c = s.branch_costs()
    if it in (0, 1, 2, 5, 10, 20, n_it - 1):
        ovf = c >= (1 << 20)
        steps = c & ((1 << 20) - 1)
        for name, sel in (("lim", limited), ("unl", ~limited)):
            o = ovf & sel
            st = steps[o]
            q = np.percentile(st, [50, 90, 99, 100]) if st.size else []
            print(f"it {it:3d} {ms[0]:.3f} ms {name}: branches {sel.sum()} lane-steps "
                  f"{steps[sel & ~ovf].sum()} overflow {o.sum()} tile-steps sum {st.sum()} "
                  f"p50/90/99/max {q}", flush=True)
