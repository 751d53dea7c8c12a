"""Synthetic-grid quality sweep on the GPU path (bit-identical to the
reference solver): generate variants, full cold-start solves, report the
reference's quality metrics.  usage: synth_explore.py '<json list of specs>'
spec = {"shape": ..., "rho": [pq, va], "kw": {generator knobs}, "seed": s}"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

arg = sys.argv[1]
specs = json.load(open(arg)) if os.path.exists(arg) else json.loads(arg)
os.makedirs("/tmp/synth_explore", exist_ok=True)
for i, sp in enumerate(specs):
    kw = sp.get("kw", {})
    seed = sp.get("seed", 2110)
    path = f"/tmp/synth_explore/v{i}.m"
    t0 = time.time()
    synth.write_case(sp["shape"], path, seed=seed, **kw)
    gen_s = time.time() - t0
    net = ga.Network(path)
    rpq, rva = sp.get("rho", [100.0, 1e4])
    extra = sp.get("cfg", {})
    cfg = ga.Config(rho_pq=rpq, rho_va=rva, **extra)
    t0 = time.time()
    st, rep = ga.solve(net, cfg)
    dt = time.time() - t0
    m = rep.metrics()
    vm, va = rep.voltages()
    out = dict(sp, status=ga.STATUS[st], time_s=round(dt, 3), gen_s=round(gen_s, 2),
               va_span=float(va.max() - va.min()), **m)
    print(json.dumps(out), flush=True)
