"""Convergence of the synthetic grids under different penalty pairs (GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case2868rte"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
for rpq, rva in [(10, 1e3), (100, 1e3), (100, 1e4), (1e3, 1e4), (1e3, 1e5), (3e3, 3e4), (3e4, 3e5)]:
    cfg = ga.Config(rho_pq=rpq, rho_va=rva, eps=eps)
    t = time.time()
    st, rep = ga.solve(net, cfg)
    m = rep.metrics()
    print(f"{shape} rho=({rpq:g},{rva:g}) {ga.STATUS[st]} inner={m['inner_iterations']:.0f} "
          f"outer={m['outer_iterations']:.0f} c_inf={m['c_inf']:.3g} obj={m['objective']:.6g} "
          f"t={time.time() - t:.1f}s", flush=True)
