"""Probe: per-branch TRON cost distribution on a synthetic shape."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_06879_b200 as ga
from paper_2110_06879_b200 import synth
shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
ex = net.export()
limited = ex["branch"][:, 5] > 0
s = ga.Session(net, ga.Config("case_ACTIVSg70k"))
for it in range(n_it):
    ms, rec = s.timed_steps(1, 0)
    c = s.branch_costs()
    if it in (0, 1, 2, 5, n_it - 1):
        for name, sel in (("lim", limited), ("unl", ~limited)):
            cc = c[sel]
            q = np.percentile(cc, [50, 90, 99, 99.9, 100])
            print(f"it {it} {ms[0]:.2f} ms {name} n={cc.size} sum={cc.sum()} mean={cc.mean():.1f} "
                  f"p50/90/99/99.9/max={q} n>=200:{(cc>=200).sum()} n>=1000:{(cc>=1000).sum()}", flush=True)
