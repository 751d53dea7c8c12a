#!/usr/bin/env python3
"""Generates tests/golden/* from the REFERENCE solver (oracle/_ref, compiled
from /root/reference/proj/src with the pinned sincos).  Run in the dev
container where /root/reference exists:

    make -C oracle && python scripts/make_golden.py

Outputs (small, committed):
  series_<case>.npz   first N inner iterations (desk config of
                      proj/tests/acceptance.cpp:58-69, max_outer=1):
                      residual series + the final AdmmState arrays
  solve_case9.json    full case9 cold-start solve: status, iteration counts,
                      quality metrics, last residual record
  sincos.npz          pinned sincos on 4096 arguments (host bits)
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import oracle  # noqa: E402

GOLDEN = os.path.join(REPO, "tests", "golden")
DESK = {
    "case9": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5),
    "case30": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5),
    "case118": dict(rho_pq=100.0, rho_va=1e4, eps=1e-6, max_inner=300),
}
ITERS = {"case9": 100, "case30": 60, "case118": 40}


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    assert oracle.have_ref(), "build oracle/_ref first (make -C oracle)"
    for name, cfg in DESK.items():
        ref = oracle.RefNet(os.path.join(REPO, "data", name + ".m"))
        n = ITERS[name]
        series, info, fin = ref.solve(**dict(cfg, max_outer=1, max_inner=n))
        keep = {k: fin[k] for k in ("x", "xbar", "z", "y", "lambda", "branch_point", "lt_ij",
                                    "lt_ji", "rho_tilde")}
        np.savez_compressed(os.path.join(GOLDEN, f"series_{name}.npz"), iters=n,
                            series=series[:, :5], **keep)
        print(name, series.shape, info[:4])
    ref = oracle.RefNet(os.path.join(REPO, "data", "case9.m"))
    series, info, _ = ref.solve(**DESK["case9"])
    out = {"status": int(info[0]), "outer_iterations": int(info[1]),
           "inner_iterations": int(info[2]), "branch_solve_failures": int(info[3]),
           "objective": info[4], "balance_inf": info[5], "limit_violation": info[6],
           "bound_violation": info[7], "c_inf": info[8],
           "last_record": [float(v) for v in series[-1, 2:5]],
           "config": DESK["case9"], "generator": "scripts/make_golden.py (reference oracle)"}
    json.dump(out, open(os.path.join(GOLDEN, "solve_case9.json"), "w"), indent=1)
    print("case9 full", out["inner_iterations"], out["objective"])
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-4 * np.pi, 4 * np.pi, 4000), [0.0, -0.0, np.pi / 4, 1e-300]])
    s, c = oracle.ref_sincos(x)
    np.savez_compressed(os.path.join(GOLDEN, "sincos.npz"), x=x, s=s, c=c)


if __name__ == "__main__":
    main()
