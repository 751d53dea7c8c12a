"""Warm-start tracking, B200 vs the reference C++ solver on all host cores
(BASELINE configs[4]): ACTIVSg25k-shaped grid, 30 snapshots
(gridcases.synth.tracking_profile), ramp_frac 0.02, the reference's preset;
gridadmm_track_run of both libraries; per-period objectives compared bit for bit.
usage: track_vs_reference.py [shape] [periods] [preset] [cpu_periods] [out.json]"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg25k"
periods = int(sys.argv[2]) if len(sys.argv) > 2 else 30
preset = sys.argv[3] if len(sys.argv) > 3 else "case_ACTIVSg25k"
cpu_periods = int(sys.argv[4]) if len(sys.argv) > 4 else periods
out_path = sys.argv[5] if len(sys.argv) > 5 else None
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
prof = synth.ensure_profile(path, periods=periods)

net = ga.Network(path)
cfg = ga.Config(preset, ramp_frac=0.02)
t0 = time.perf_counter()
st, trk = ga.track(net, cfg, prof)
gpu_wall = time.perf_counter() - t0
gper = trk.period_table()
gobj = [trk.period_report(p + 1).metric("objective") for p in range(len(gper))]

cpu_prof = prof
if cpu_periods < periods:  # the first cpu_periods snapshots of the same profile
    cpu_prof = prof[:-4] + f"_first{cpu_periods}.csv"
    with open(prof) as f, open(cpu_prof, "w") as g:
        for ln in f:
            if ln.startswith("period") or int(ln.split(",", 1)[0]) <= cpu_periods:
                g.write(ln)
workers = os.cpu_count() or 1
t1 = time.perf_counter()
rst, rper = oracle.ref_track(path, cpu_prof, preset, ramp_frac=0.02, workers=workers)
cpu_wall = time.perf_counter() - t1
h = oracle.ref_capi()
# per-period solve seconds of the reference come from its periods.csv
rtimes = [p.get("time_s") for p in rper]
same = [float(gobj[i]).hex() == float(rper[i]["objective"]).hex() for i in range(len(rper))]
gwarm = [p["time_s"] for p in gper[1:]]
cwarm = [t for t in rtimes[1:] if t is not None]
out = {"shape": shape, "periods": periods, "preset": preset, "ramp_frac": 0.02,
       "gpu_status": ga.STATUS[st], "gpu_wall_s": gpu_wall, "gpu_cold_s": gper[0]["time_s"],
       "gpu_warm_s_per_step_mean": float(np.mean(gwarm)), "gpu_warm_s_per_step_max": float(np.max(gwarm)),
       "gpu_warm_inner_mean": float(np.mean([p["inner"] for p in gper[1:]])),
       "gpu_c_inf_max": float(max(p["c_inf"] for p in gper)),
       "cpu_status": ga.STATUS[rst], "cpu_periods": len(rper), "cpu_wall_s": cpu_wall,
       "cpu_cores": workers, "cpu_cold_s": rtimes[0],
       "cpu_warm_s_per_step_mean": float(np.mean(cwarm)) if cwarm else None,
       "gpu_warm_s_per_step_mean_same_periods": float(np.mean(gwarm[:len(cwarm)])) if cwarm else None,
       "warm_speedup_same_periods": (float(np.mean(cwarm)) / float(np.mean(gwarm[:len(cwarm)]))
                                     if cwarm else None),
       "cpu_inner_per_period": [p.get("inner_iterations") for p in rper],
       "objectives_bit_identical": all(same), "periods_compared": len(same),
       "gpu_per_period": gper}
print(json.dumps(out), flush=True)
if out_path:
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
