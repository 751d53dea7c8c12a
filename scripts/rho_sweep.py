"""Convergence of the synthetic grids under different penalty pairs (GPU).
usage: rho_sweep.py <shape> <eps> <max_inner> <max_outer> [rho_pq:rho_va ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case2868rte"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
max_inner = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
max_outer = int(sys.argv[4]) if len(sys.argv) > 4 else 20
pairs = [tuple(map(float, a.split(":"))) for a in sys.argv[5:]] or [
    (10, 1e3), (100, 1e3), (100, 1e4), (1e3, 1e4), (1e3, 1e5), (3e3, 3e4), (3e4, 3e5)]
net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
for rpq, rva in pairs:
    cfg = ga.Config(rho_pq=rpq, rho_va=rva, eps=eps, max_inner=max_inner, max_outer=max_outer)
    t = time.time()
    st, rep = ga.solve(net, cfg)
    m = rep.metrics()
    dt = time.time() - t
    print(f"{shape} rho=({rpq:g},{rva:g}) {ga.STATUS[st]} inner={m['inner_iterations']:.0f} "
          f"outer={m['outer_iterations']:.0f} c_inf={m['c_inf']:.3g} obj={m['objective']:.8g} "
          f"t={dt:.1f}s it/s={m['inner_iterations'] / dt:.0f}", flush=True)
