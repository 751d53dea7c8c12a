"""Probe: kernel breakdown and TRON cost distribution deep into a solve
(after `skip` inner iterations of outer iteration 1, or after full outer
iterations via the C-ABI solve semantics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case118"
outers = int(sys.argv[3]) if len(sys.argv) > 3 else 5
p = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(p)
ex = net.export()
limited = ex["branch"][:, 5] > 0
s = ga.Session(net, ga.Config(preset))
for o in range(outers):
    rec, stop = s.iterate(1000)
    z = float(rec[-1, 2])
    st = s.get_state()
    prev = -1.0 if o == 0 else prev_z
    s.phase("outer", z, prev)
    prev_z = z
    c0 = s.step_counters()
    k0 = [s.kernel_time(c) for c in range(4)]
    ms, _ = s.timed_steps(5, 0)
    c1 = s.step_counters()
    k1 = [s.kernel_time(c) for c in range(4)]
    c = s.branch_costs()
    print(f"outer {o + 1}: beta={st['beta'][0]:.3g} step ms {np.round(ms, 3)} "
          f"kernels/5 {[round((k1[i][0] - k0[i][0]) / 5, 3) for i in range(4)]} "
          f"tron(ref) {[c1[i] - c0[i] for i in (0, 1)]} exec {[c1[i] - c0[i] for i in (2, 3)]}",
          flush=True)
    lib_name = os.environ.get("GRIDADMM_LIB", "")
    stats_build = "stats" in lib_name or "steps" in lib_name
    for name, sel in (("lim", limited), ("unl", ~limited)):
        cc = c[sel]
        if stats_build:  # br_cost = executed steps (+2^20 when the tile phase ran it)
            ovf = cc >= (1 << 20)
            stp = cc & ((1 << 20) - 1)
            t = stp[ovf]
            print(f"   {name}: lane-only {(~ovf).sum()} steps {stp[~ovf].sum()} | overflow {ovf.sum()} "
                  f"steps {t.sum()} p50/90/99/max {np.percentile(t, [50, 90, 99, 100]) if t.size else []}",
                  flush=True)
        else:
            print(f"   {name}: mean {cc.mean():.1f} p50/90/99/max {np.percentile(cc, [50, 90, 99, 100])} "
                  f"n>=200 {(cc >= 200).sum()} n>=1000 {(cc >= 1000).sum()}", flush=True)
