"""ncu target: N inner iterations of the 70k-shaped cold start (no timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
s = ga.Session(net, ga.Config("case_ACTIVSg70k"))
s.iterate(n_it)
