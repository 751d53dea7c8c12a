"""Late-solve window, GPU vs the reference CPU solver on the same state.

Runs the 70k-shaped cold start on the device (driver.cpp:152-239 replica:
inner loops of max_inner, outer updates with the beta schedule) up to the
start of outer iteration `outer`, downloads the full AdmmState, then times
K further inner iterations (a) on the device (CUDA events) and (b) with the
reference C++ solver (oracle/_ref, all host cores) warm-started from that
state, and checks that both produce bit-identical residual series.
usage: late_window_compare.py [shape] [rho_pq] [rho_va] [outer] [K]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
rpq = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
rva = float(sys.argv[3]) if len(sys.argv) > 3 else 1e4
outer = int(sys.argv[4]) if len(sys.argv) > 4 else 10
K = int(sys.argv[5]) if len(sys.argv) > 5 else 5
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(path)
cfg = ga.Config(rho_pq=rpq, rho_va=rva)
s = ga.Session(net, cfg)
prev = -1.0
t0 = time.perf_counter()
done = 0
for o in range(outer - 1):
    rec, _ = s.iterate(1000)
    done += len(rec)
    z = float(rec[-1, 2])
    s.phase("outer", z, prev)
    prev = z
t_reach = time.perf_counter() - t0
st = s.get_state()
ms, rec = s.timed_steps(K, 0)
workers = os.cpu_count() or 1
ref = oracle.RefNet(path)
t1 = time.perf_counter()
series, info, _ = ref.solve(init=st, rho_pq=rpq, rho_va=rva, max_outer=1, max_inner=K, workers=workers)
cpu_wall = time.perf_counter() - t1
el = series[:, 5]
cpu_ms = np.diff(np.concatenate([[0.0], el])) * 1e3
same = bool(np.array_equal(series[:K, 2:5].view(np.uint64), rec[:K, 0:3].view(np.uint64)))
out = {"shape": shape, "rho": [rpq, rva], "start_iteration": done, "beta": float(st["beta"][0]),
       "gpu_reach_s": t_reach, "K": K, "gpu_ms_per_iter": [round(float(x), 3) for x in ms],
       "cpu_ms_per_iter": [round(float(x), 1) for x in cpu_ms], "cpu_workers": workers,
       "gpu_iters_per_s": K / (float(np.sum(ms)) * 1e-3),
       "cpu_iters_per_s": K / float(el[-1]) if el[-1] > 0 else None,
       "residuals_bit_identical": same}
out["ratio"] = out["gpu_iters_per_s"] / out["cpu_iters_per_s"] if out["cpu_iters_per_s"] else None
print(json.dumps(out), flush=True)
