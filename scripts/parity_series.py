"""Residual-series parity at scale: two device runs (determinism) and the
reference solver, first N inner iterations of a cold start.
usage: parity_series.py [shape] [preset] [N] [timed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case_ACTIVSg70k"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 35
timed = len(sys.argv) > 4 and sys.argv[4] == "timed"
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(path)
cfg = ga.Config(preset)
runs = []
for r in range(3):
    s = ga.Session(net, cfg)
    if timed:
        _, a = s.timed_steps(5, 0)
        _, b = s.timed_steps(N - 5, 256 << 20)
        rec = np.concatenate([a, b])
    else:
        rec, _ = s.iterate(N)
    runs.append(rec[:, 0:3].copy())
    s.close()
ref = oracle.RefNet(path)
series, _, _ = ref.solve(rho_pq=cfg["rho_pq"], rho_va=cfg["rho_va"], max_outer=1, max_inner=N,
                         workers=os.cpu_count() or 1)
want = series[:, 2:5]
for r, got in enumerate(runs):
    ne = np.nonzero(got.view(np.uint64) != want.view(np.uint64))
    if ne[0].size:
        i, c = ne[0][0], ne[1][0]
        print(f"run {r}: first mismatch iteration {i} column {c}: gpu {got[i, c]!r} ref {want[i, c]!r}; "
              f"{ne[0].size} entries differ")
    else:
        print(f"run {r}: bit-identical over {N} iterations")
