import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2110_06879_b200 as ga
for name in ["case9", "case30", "case118"]:
    net = ga.Network(f"data/{name}.m")
    cfg = ga.Config(rho_pq=100, rho_va=1e4, eps=1e-5)
    s = ga.Session(net, cfg)
    t = time.time(); rec, stop = s.iterate(200); dt = time.time() - t
    print(name, "200 its", round(dt, 4), "s", [s.kernel_time(k) for k in range(4)], s.counters(), flush=True)
