"""Probe: 70k-shaped synthetic case on the GPU — per-iteration kernel times,
TRON iteration counts and residual trend over the first iterations."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_06879_b200 as ga
from paper_2110_06879_b200 import synth
shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case_ACTIVSg70k"
n_it = int(sys.argv[3]) if len(sys.argv) > 3 else 50
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
cfg = ga.Config(preset)
s = ga.Session(net, cfg)
t = time.time()
ms, rec = s.timed_steps(n_it, 0)
print(shape, preset, "wall", round(time.time() - t, 3), "s for", n_it)
print("step ms first/median/last", ms[:3], np.median(ms), ms[-3:])
print("kernels", [s.kernel_time(c) for c in range(4)], "tron iters (4,6)", s.counters())
for k in list(range(0, n_it, max(1, n_it // 10))) + [n_it - 1]:
    print(k, rec[k])
print("fp64 peak", ga.fp64_peak(0))
