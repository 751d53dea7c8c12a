"""Time-to-converge, B200 vs the reference C++ solver on all host cores, same
synthetic case and penalty, full cold-start solves (BASELINE config[1]).
Both runs must produce the same iteration count and objective bits.
usage: converge_vs_reference.py <shape> [rho_pq] [rho_va]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case2868rte"
rpq = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
rva = float(sys.argv[3]) if len(sys.argv) > 3 else 1e4
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(path)
cfg = ga.Config(rho_pq=rpq, rho_va=rva)
ga.solve(net, ga.Config(rho_pq=rpq, rho_va=rva, max_outer=1, max_inner=2))  # context / modules
t0 = time.perf_counter()
st, rep = ga.solve(net, cfg)
gpu_s = time.perf_counter() - t0
m = rep.metrics()
workers = os.cpu_count() or 1
ref = oracle.RefNet(path)
t1 = time.perf_counter()
series, info, _ = ref.solve(rho_pq=rpq, rho_va=rva, workers=workers)
cpu_s = time.perf_counter() - t1
print("gpu", gpu_s, m["inner_iterations"], m["objective"], "cpu", cpu_s, info[2], info[4], flush=True)
out = {"shape": shape, "rho": [rpq, rva], "gpu_status": ga.STATUS[st], "gpu_time_s": gpu_s,
       "gpu_inner": m["inner_iterations"], "gpu_objective": m["objective"], "gpu_c_inf": m["c_inf"],
       "cpu_time_s": cpu_s, "cpu_cores": workers, "cpu_inner": float(info[2]),
       "cpu_objective": float(info[4]),
       "same_iterations": bool(m["inner_iterations"] == info[2]),
       "objective_bit_identical": bool(np.float64(m["objective"]).view(np.uint64) ==
                                       np.float64(info[4]).view(np.uint64)),
       "speedup": cpu_s / gpu_s}
print(json.dumps(out), flush=True)
