"""Time-to-converge on a synthetic shape: the B200 solver through the C ABI
(gridadmm_solve) and the reference solver (oracle/_ref, all host threads) on
the same case and config.  Both run the identical (bit-exact) trajectory, so
iteration counts must match.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
import oracle  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case118"
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
run_cpu = (sys.argv[4] if len(sys.argv) > 4 else "1") == "1"
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(path)
cfg = ga.Config(preset, eps=eps)
t = time.perf_counter()
st, rep = ga.solve(net, cfg)
t_gpu = time.perf_counter() - t
out = {"shape": shape, "preset": preset, "eps": eps, "gpu_status": ga.STATUS[st],
       "gpu_time_s": t_gpu, "gpu": rep.metrics()}
print(json.dumps(out), flush=True)
if run_cpu:
    workers = os.cpu_count() or 1
    ref = oracle.RefNet(path)
    t = time.perf_counter()
    series, info, _ = ref.solve(rho_pq=cfg["rho_pq"], rho_va=cfg["rho_va"], eps=eps,
                                workers=workers)
    t_cpu = time.perf_counter() - t
    out.update({"cpu_time_s": t_cpu, "cpu_workers": workers, "cpu_status": int(info[0]),
                "cpu_inner": int(info[2]), "cpu_outer": int(info[1]), "cpu_objective": float(info[4]),
                "same_iterations": bool(int(info[2]) == int(out["gpu"]["inner_iterations"])),
                "same_objective_bits": bool(float(info[4]) == float(out["gpu"]["objective"]))})
    print(json.dumps(out), flush=True)
