"""Lean FP64 op census of the C restatement (oracle/gridadmm_oracle.c FL())
over inner iterations W..W+K-1 of a cold start: flops per reference TRON
iteration for 4- and 6-variable branches (the bench roofline numerator).
usage: census_window.py <case.m> <W> <K> [preset]"""
import sys, time, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle
path, W, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rpq, rva = oracle.ref_preset(sys.argv[4]) if len(sys.argv) > 4 else (3e4, 3e5)
p = oracle.PortNet(path)
t = time.time()
s1, info, st = p.solve(rho_pq=rpq, rho_va=rva, max_outer=1, max_inner=W)
c0 = p.census(reset=True)
s2, info, st2 = p.solve(init=st, rho_pq=rpq, rho_va=rva, max_outer=1, max_inner=K)
c = p.census(reset=True)
print(json.dumps({"path": path, "window": [W, W + K - 1], "rho": [rpq, rva], "flops": c[0], "iters4": c[1], "iters6": c[2], "flops4": c[3], "flops6": c[4], "sincos": c[5],
  "per_iter4": c[3] / max(1, c[1]), "per_iter6": c[4] / max(1, c[2]), "time_s": time.time() - t}))
