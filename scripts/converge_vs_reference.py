"""Time-to-converge, B200 vs the reference C++ solver on all host cores: the
same synthetic case, the reference's preset penalties and default
tolerances, full cold-start solves through each library's gridadmm_solve
(BASELINE configs[1], [3]).  Both runs must give the same iteration count
and objective bits.
usage: converge_vs_reference.py <shape> <preset|rho_pq:rho_va> [eps] [out.json]"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case_ACTIVSg70k"
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
out_path = sys.argv[4] if len(sys.argv) > 4 else None
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
if ":" in preset:
    rpq, rva = (float(v) for v in preset.split(":"))
else:
    rpq, rva = oracle.ref_preset(preset)
settings = dict(rho_pq=rpq, rho_va=rva, eps=eps)

net = ga.Network(path)
ga.solve(net, ga.Config(**settings, max_outer=1, max_inner=2))  # CUDA context / modules
t0 = time.perf_counter()
st, rep = ga.solve(net, ga.Config(**settings))
gpu_s = time.perf_counter() - t0
m = rep.metrics()

workers = os.cpu_count() or 1
h = oracle.ref_capi()
rnet = ctypes.c_void_p()
assert h.gridadmm_network_load(os.fsencode(path), ctypes.byref(rnet)) == 0
c = h.gridadmm_config_new()
for k, v in dict(settings, workers=workers).items():
    assert h.gridadmm_config_set(c, k.encode(), float(v)) == 0, k
rrep = ctypes.c_void_p()
t1 = time.perf_counter()
rst = h.gridadmm_solve(rnet, c, ctypes.byref(rrep))
cpu_s = time.perf_counter() - t1
rm = oracle.ref_metrics(h, rrep)
out = {"shape": shape, "preset": preset, "rho": [rpq, rva], "eps": eps,
       "gpu_status": ga.STATUS[st], "gpu_time_s": gpu_s, "gpu_inner": m["inner_iterations"],
       "gpu_outer": m["outer_iterations"], "gpu_objective": m["objective"],
       "gpu_c_inf": m["c_inf"], "cpu_status": ga.STATUS[rst], "cpu_time_s": cpu_s,
       "cpu_cores": workers, "cpu_inner": rm["inner_iterations"], "cpu_objective": rm["objective"],
       "cpu_objective_hex": float(rm["objective"]).hex(), "cpu_c_inf": rm["c_inf"],
       "same_iterations": m["inner_iterations"] == rm["inner_iterations"],
       "objective_bit_identical": float(m["objective"]).hex() == float(rm["objective"]).hex(),
       "c_inf_bit_identical": float(m["c_inf"]).hex() == float(rm["c_inf"]).hex(),
       "speedup": cpu_s / gpu_s}
print(json.dumps(out), flush=True)
if out_path:
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
