"""Probe (debug build, GRIDADMM_LIB=.../libgridadmm_stats.so): TRON path
statistics per step over one ADMM iteration of a synthetic shape."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
s = ga.Session(net, ga.Config("case_ACTIVSg70k"))
buf = (ctypes.c_ulonglong * 8)()
s.timed_steps(n_it - 1, 0)
ga.lib().gridadmm_debug_tron_stats(buf, 1)
ms, _ = s.timed_steps(1, 0)
ga.lib().gridadmm_debug_tron_stats(buf, 1)
st = list(buf)
names = ["steps", "cauchy_extrap", "cauchy_halve", "cg_iters", "ls_steps", "chol_fail", "rejected", "iter>=100"]
print("iteration", n_it - 1, "ms", ms[0])
for k, nm in enumerate(names):
    print(f"{nm:14s} {st[k]:12d}  per step {st[k] / max(1, st[0]):.3f}")
