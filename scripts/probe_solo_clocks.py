"""Probe (clock build, GRIDADMM_LIB=.../libgridadmm_clk.so): cycles per TRON
step section for whole-warp (T=32) solves, late in a solve where the solo
phase runs.  Sections: 0 gradient, 1 Hessian, 2 Cauchy, 3 CG, 4 line search
+ trial point, 5 value, 6 ratio/update."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
outers = int(sys.argv[2]) if len(sys.argv) > 2 else 9
net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
s = ga.Session(net, ga.Config("case118"))
prev = -1.0
for o in range(outers):
    rec, _ = s.iterate(1000)
    z = float(rec[-1, 2])
    s.phase("outer", z, prev)
    prev = z
buf = (ctypes.c_ulonglong * 8)()
ga.lib().gridadmm_debug_tron_stats(buf, 1)
c0 = s.step_counters()
ms, _ = s.timed_steps(5, 0)
ga.lib().gridadmm_debug_tron_stats(buf, 1)
c = s.branch_costs()
solo_steps = None
names = ["gradient", "hessian", "cauchy", "cg", "linesearch", "value", "update"]
tot = sum(buf[k] for k in range(7))
print("step ms", np.round(ms, 3), "max branch steps", int((c & ((1 << 20) - 1)).max()), "T=32 steps", buf[7], "cycles/step", round(tot / max(1, buf[7])))
for k, nm in enumerate(names):
    print(f"{nm:10s} {buf[k]:14d} cycles ({100 * buf[k] / max(1, tot):5.1f}%)")
