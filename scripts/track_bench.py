"""Warm-start tracking benchmark (BASELINE config[4]): an ACTIVSg25k-shaped
synthetic grid over a 30-snapshot load sequence — per-bus multipliers
m_{t,i} = P(t) (1 + eps_{t,i}), P(t) a linear interpolation of a smooth
series spanning <= 5%, eps ~ N(0, 0.005^2), seeded;
ramp_frac 0.02.  Runs gridadmm_track_run (the reference's tracking entry
point, C ABI) and prints one JSON line with seconds per snapshot."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402


def write_profile(net, periods, path, seed=25, swing=0.05, noise=0.005):
    rng = np.random.default_rng(seed)
    ids = net.export()["bus_id"]
    hourly = 1.0 + swing * np.sin(np.linspace(0.0, np.pi, 4))  # <= 5% swing
    t = np.linspace(0, len(hourly) - 1, periods)
    level = np.interp(t, np.arange(len(hourly)), hourly) / hourly[0]
    with open(path, "w") as f:
        f.write("period,bus,multiplier\n")
        for p in range(periods):
            m = level[p] * (1.0 + noise * rng.standard_normal(len(ids)))
            f.write("".join(f"{p + 1},{i},{v:.9f}\n" for i, v in zip(ids, m)))
    return path


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg25k"
    periods = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    preset = sys.argv[3] if len(sys.argv) > 3 else "case_ACTIVSg25k"  # or "rho_pq:rho_va"
    max_inner = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
    max_outer = int(sys.argv[5]) if len(sys.argv) > 5 else 20
    swing = float(sys.argv[6]) if len(sys.argv) > 6 else 0.05
    noise = float(sys.argv[7]) if len(sys.argv) > 7 else 0.005
    path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
    net = ga.Network(path)
    prof = write_profile(net, periods, f"/tmp/gridadmm_cases/{shape}_profile_{periods}.csv",
                         swing=swing, noise=noise)
    if ":" in preset:
        rpq, rva = (float(v) for v in preset.split(":"))
        cfg = ga.Config(rho_pq=rpq, rho_va=rva, max_inner=max_inner, max_outer=max_outer,
                        ramp_frac=0.02)
    else:
        cfg = ga.Config(preset, max_inner=max_inner, max_outer=max_outer, ramp_frac=0.02)
    t0 = time.perf_counter()
    st, trk = ga.track(net, cfg, prof)
    wall = time.perf_counter() - t0
    per = []
    tmp = f"/tmp/gridadmm_cases/{shape}_periods.csv"
    trk.write_periods(tmp)
    rows = np.genfromtxt(tmp, delimiter=",", names=True)
    for r in np.atleast_1d(rows):
        per.append({"period": int(r["period"]), "inner": int(r["inner_iters"]),
                    "time_s": float(r["time_s"]), "c_inf": float(r["viol_inf"])})
    warm = [p["time_s"] for p in per[1:]]
    out = {"shape": shape, "periods": periods, "preset": preset, "swing": swing, "noise": noise,
           "status": ga.STATUS[st],
           "wall_s": wall, "cold_s": per[0]["time_s"] if per else None,
           "warm_s_per_step_mean": float(np.mean(warm)) if warm else None,
           "warm_s_per_step_max": float(np.max(warm)) if warm else None,
           "warm_inner_mean": float(np.mean([p["inner"] for p in per[1:]])) if len(per) > 1 else None,
           "per_period": per}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
