"""TRON path statistics over an iteration window (debug build with
-DGA_TRON_STATS: `make -C paper_2110_06879_b200/csrc stats`, then run with
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so).
usage: probe_path_stats.py <shape> <preset> <warmup> <window>"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_06879_b200 as ga  # noqa: E402
from gridcases import synth  # noqa: E402

shape, preset = sys.argv[1], sys.argv[2]
warm, window = int(sys.argv[3]), int(sys.argv[4])
net = ga.Network(synth.ensure_case(shape, "/tmp/gridadmm_cases"))
s = ga.Session(net, ga.Config(preset))
s.iterate(warm)
buf = (ctypes.c_ulonglong * 8)()
ga.lib().gridadmm_debug_tron_stats(buf, 1)
c0 = s.step_counters()
s.iterate(window)
ga.lib().gridadmm_debug_tron_stats(buf, 1)
c1 = s.step_counters()
names = ["steps", "cauchy_extrapolations", "cauchy_halvings", "cg_iterations", "line_search_trials",
         "chol_fail_or_fixed_point", "rejected_steps", "steps_iter_ge_100"]
st = dict(zip(names, list(buf)))
steps = max(1, st["steps"])
out = {"shape": shape, "preset": preset, "window": [warm, warm + window - 1],
       "step_counters_delta": [int(b - a) for a, b in zip(c0, c1)], "totals": st,
       "per_step": {k: v / steps for k, v in st.items()}}
print(json.dumps(out))
