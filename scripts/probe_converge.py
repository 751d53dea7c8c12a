"""Probe: full cold-start solve of a synthetic shape through the C ABI; prints
status, iterations, time, quality and per-100-iteration residuals."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case_ACTIVSg70k"
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
max_inner = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
cfg = ga.Config(preset, eps=eps, max_inner=max_inner)
t = time.time()
st, rep = ga.solve(net, cfg)
dt = time.time() - t
m = rep.metrics()
print(f"{shape} preset={preset} eps={eps} status={ga.STATUS[st]} time={dt:.2f}s "
      f"its/s={m['inner_iterations'] / dt:.1f}", m, flush=True)
out = f"/tmp/conv_{shape}_{preset}.csv"
rep.write_convergence(out)
rows = np.loadtxt(out, delimiter=",", skiprows=1)
for k in list(range(0, len(rows), max(1, len(rows) // 25))) + [len(rows) - 1]:
    print("  ", rows[k][:5])
