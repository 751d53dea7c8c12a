"""Parity at scale: phase replay on a synthetic grid (device vs reference
oracle, bit-exact), reporting the first mismatching phase/field/index.
usage: parity_70k.py [shape] [preset] [iterations]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2110_06879_b200 as ga  # noqa: E402
from paper_2110_06879_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "case_ACTIVSg70k"
preset = sys.argv[2] if len(sys.argv) > 2 else "case_ACTIVSg70k"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 6
FIELDS = ("x", "xbar", "z", "y", "lambda", "rho", "bus_w", "bus_theta", "branch_point", "lt_ij",
          "lt_ji", "rho_tilde", "beta")
path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
net = ga.Network(path)
cfg = ga.Config(preset)
d = dict(rho_pq=cfg["rho_pq"], rho_va=cfg["rho_va"], workers=os.cpu_count() or 1)
sess = ga.Session(net, cfg)
ref = oracle.RefNet(path)
s = ref.cold_start(**d)


def diff(gpu, ref_s, where):
    bad = False
    for f in FIELDS:
        a = np.ascontiguousarray(gpu[f], dtype=np.float64).view(np.uint64)
        b = np.ascontiguousarray(ref_s[f], dtype=np.float64).view(np.uint64)
        if not np.array_equal(a, b):
            idx = np.nonzero(a != b)[0]
            print(f"MISMATCH {where} {f}: {idx.size} of {a.size}, first {idx[:8].tolist()} "
                  f"gpu {np.asarray(gpu[f]).ravel()[idx[0]]!r} ref {np.asarray(ref_s[f]).ravel()[idx[0]]!r}",
                  flush=True)
            bad = True
    return bad


diff(sess.get_state(), s, "cold start")
for it in range(iters):
    for p in ["generators", "branches", "buses", "z", "y"]:
        sess.set_state(s)
        sess.phase(p)
        ref.phase(ga.PHASES[p], s, **d)
        if diff(sess.get_state(), s, f"it {it} phase {p}"):
            sys.exit(1)
    print(f"it {it} ok", flush=True)
# fused iteration path vs the replayed reference state
sess.set_state(s)
rec, _ = sess.iterate(3)
series, _, _ = ref.solve(init=s, max_outer=1, max_inner=3, **d)
print("fused iterate bit-identical:",
      bool(np.array_equal(series[:3, 2:5].view(np.uint64), rec[:3, 0:3].view(np.uint64))))
