#!/usr/bin/env python3
"""bench.py — ADMM iterations/s and time-to-converge of the B200-native
gridadmm on an ACTIVSg70k-shaped grid (BASELINE.json metric, configs[3]),
with the reference C++ solver timed on the same host.

A "step" is one inner ADMM iteration of the two-level ADMM over the whole
grid: generator projection -> branch NLPs -> bus consensus -> z / y /
residual norms, plus the host's read of the norms that drive the loop
control (proj/src/driver.cpp:155-186).  The first W iterations from the cold
start are the warm-up, the next K are timed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Both arms run the same workload (WORKLOAD below, one shared `config` dict):
the seeded synthetic ACTIVSg70k-shaped case (gridcases/synth.py: exactly the
published 70,000 buses / 10,390 generators / 88,207 branches) with the
reference's own preset for ACTIVSg70k (rho_pq 3e4, rho_va 3e5; capi.cpp:36)
and its default tolerances (eps 1e-4, 20 x 1000 iterations).

* `value`: K x ranks / max-over-ranks device time of the K steps, state
  resident in HBM, each step timed with CUDA events on the solver's stream,
  L2 flushed (256 MiB write) between steps outside the events.
* `e2e`: the same iterations through the public C ABI with host buffers:
  gridadmm_solve(max_outer 1, max_inner W+K) on a loaded network (network
  upload, device cold start, every iteration's norm readback, solution
  download inside the wall-clock region).
* `converge`: time-to-converge of the full cold start through gridadmm_solve
  (the reference's stop rules), with the reference's quality metrics (c_inf,
  objective) of the result; `cpu_full_solve_s` is the reference's own full
  solve of the same case on a box of this pool, measured once
  (profiles/r02_converge_vs_reference_70k.json) because it runs ~30 minutes.
* `track`: warm-start tracking, ACTIVSg25k-shaped, 30 snapshots
  (BASELINE.json configs[4]), seconds per warm snapshot.
* `roofline`: the branch-NLP kernels (dominant) against the measured FP64
  DMUL+DADD peak (the kernels are built -fmad=false for bit-exactness); the
  flop count is the lean op census of the C restatement on this workload.
* `cpu_baseline`: the reference C++ solver (oracle/_ref, compiled unmodified
  from the reference sources) through its own C ABI on all host cores,
  timing a bounded sample of the SAME iterations (trajectory bit-identical).
* `--impl reference`: that reference solver alone (rank 0), same metric,
  same config; it imports only oracle/ and gridcases/, never the product.

Multi-GPU (torchrun, N>1): the grid is split over the N GPUs by the
bus-graph partition with NCCL boundary exchange (strong scaling).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

# the library splits the bus kernel around the tile phase unless disabled
BUS_OVERLAP = os.environ.get("GRIDADMM_BUS_OVERLAP", "1") != "0"
SOLO = False  # set from the config (tile_budget > 0)

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ADMM iters/sec & time-to-converge (s) on ACTIVSg70k; warm-start track s/step"
DATA = "synthetic (gridcases.synth v2: seeded case30/case118 tiling to ACTIVSg70k dims)"
L2_FLUSH_BYTES = 256 << 20
WORKLOAD = {"shape": "case_ACTIVSg70k", "seed": 2110, "preset": "case_ACTIVSg70k"}
# Lean FP64 op census per reference TRON iteration (flops whose results are
# consumed: branch evaluation + TRON core, amortized per-branch setup), from
# the C restatement's counters (oracle/gridadmm_oracle.c FL()) on THIS
# workload (profiles/r02_census_70k_window.json overrides these fallbacks).
CENSUS_FLOPS = {4: 1529.5, 6: 3296.6}
CENSUS_FILE = os.path.join(REPO, "profiles", "r02_census_70k_window.json")
CPU_FULL_SOLVE_FILE = os.path.join(REPO, "profiles", "r02_converge_vs_reference_70k.json")
TRACK_CPU_FILE = os.path.join(REPO, "profiles", "r02_track_25k_vs_reference.json")
NCU_TRAFFIC_FILE = os.path.join(REPO, "profiles", "r02_ncu_traffic.jsonl")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--cpu-steps", type=int, default=10, help="timed iterations of the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-converge", action="store_true",
                    help="skip the time-to-converge run (full cold-start solve)")
    ap.add_argument("--no-track", action="store_true", help="skip the warm-start tracking run")
    return ap.parse_args()


def workload_config(args, dims):
    """The `config` object both arms print (identical by construction)."""
    nb, ng, nl = dims
    w = WORKLOAD
    return {"workload": f"{w['shape']}-shaped synthetic grid ({nb} buses, {ng} gens, {nl} "
                        f"branches, m={2 * ng + 8 * nl}) cold start, preset {w['preset']}, "
                        f"inner iterations {args.warmup}..{args.warmup + args.steps - 1}",
            "shape": w["shape"], "seed": w["seed"], "preset": w["preset"],
            "l2": "GPU arm: L2 flushed between timed steps by a 256 MiB write outside the "
                  "timed events (state + network ~57 MB)"}


class Dist:
    """Host-side plumbing between ranks (gloo): barriers, the NCCL unique id
    broadcast, max-over-ranks of device times.  The solver's own data path
    between GPUs is NCCL inside libgridadmm (gridadmm_session_new_dist)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            import torch
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist
            self.torch = torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def bcast(self, obj):
        if self.world == 1:
            return obj
        box = [obj]
        self.dist.broadcast_object_list(box, src=0)
        return box[0]

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def case_file(d: Dist) -> str:
    from gridcases import synth
    directory = os.path.join("/tmp", "gridadmm_cases")
    path = synth.case_path(WORKLOAD["shape"], directory, seed=WORKLOAD["seed"])
    if d.rank == 0:
        synth.ensure_case(WORKLOAD["shape"], directory, seed=WORKLOAD["seed"])
    d.barrier()
    while not os.path.exists(path):  # ranks on the same host share /tmp
        time.sleep(0.2)
    return path


def _load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# reference arm: the unmodified reference solver through its own C ABI
# ---------------------------------------------------------------------------

def reference_run(path: str, warmup: int, steps: int, workers: int):
    """gridadmm_solve of the reference library (oracle/_ref) with the preset
    from its own table, max_outer 1, max_inner W+K, `workers` host threads;
    iterations/s over iterations W..W+K-1 from the elapsed_s column of its
    own convergence.csv (outputs.cpp:110-120).  Returns (rate, dt, wall,
    series[n, 6], dims)."""
    import oracle
    if not oracle.have_ref():
        raise RuntimeError("oracle/_ref/libgridadmm_ref.so missing")
    h = oracle.ref_capi()
    net = ctypes.c_void_p()
    if h.gridadmm_network_load(os.fsencode(path), ctypes.byref(net)) != 0:
        raise RuntimeError(h.gridadmm_last_error().decode())
    dims = (h.gridadmm_network_num_buses(net), h.gridadmm_network_num_generators(net),
            h.gridadmm_network_num_branches(net))
    c = h.gridadmm_config_new()
    assert h.gridadmm_config_preset(c, WORKLOAD["preset"].encode()) == 0
    for k, v in (("max_outer", 1), ("max_inner", warmup + steps), ("workers", workers)):
        assert h.gridadmm_config_set(c, k.encode(), float(v)) == 0, k
    rep = ctypes.c_void_p()
    t0 = time.perf_counter()
    st = h.gridadmm_solve(net, c, ctypes.byref(rep))
    wall = time.perf_counter() - t0
    if st not in (0, 4):
        raise RuntimeError(f"reference solve status {st}: {h.gridadmm_last_error().decode()}")
    with tempfile.TemporaryDirectory() as td:
        csv = os.path.join(td, "convergence.csv")
        assert h.gridadmm_report_write_convergence(rep, os.fsencode(csv)) == 0
        series = np.loadtxt(csv, delimiter=",", skiprows=1, ndmin=2)
    h.gridadmm_report_free(rep)
    h.gridadmm_config_free(c)
    h.gridadmm_network_free(net)
    el = series[:, 5]
    start = el[warmup - 1] if warmup > 0 else 0.0
    dt = float(el[warmup + steps - 1] - start)
    return steps / dt, dt, wall, series, dims


def run_reference_arm(args, d: Dist):
    if d.rank != 0:
        return
    from gridcases import synth
    path = synth.ensure_case(WORKLOAD["shape"], "/tmp/gridadmm_cases", seed=WORKLOAD["seed"])
    workers = os.cpu_count() or 1
    rate, dt, wall, _, dims = reference_run(path, args.warmup, args.steps, workers)
    sample = (f"inner iterations {args.warmup}..{args.warmup + args.steps - 1} of the cold "
              f"start, reference C++ solver (oracle/_ref, unmodified sources) via its C ABI, "
              f"workers={workers}; {dt:.1f} s of {wall:.1f} s wall")
    line = {
        "metric": METRIC, "impl": "reference", "value": rate, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(args, dims),
        "cpu_baseline": {"value": rate, "unit": "iters/s", "cores": workers, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200_partitioned(args, d: Dist, ga, net):
    """N > 1: one grid split over N GPUs by the bus-graph partition (strong
    scaling); every step is one ADMM iteration of the whole grid, boundary
    rows and residual norms exchanged with NCCL inside the library.  Device
    time per step from CUDA events on each rank's stream, max over ranks."""
    dev = d.local
    cfg = ga.Config(WORKLOAD["preset"], device=dev)
    nccl_id = d.bcast(ga.nccl_unique_id() if d.rank == 0 else None)
    sess = ga.Session.distributed(net, cfg, d.rank, d.world, nccl_id)
    sess.timed_steps(args.warmup, 0)
    d.barrier()
    with ClockSampler(dev) as clk:
        step_ms, rec = sess.timed_steps(args.steps, L2_FLUSH_BYTES)
    d.barrier()
    max_ms = d.max(float(np.sum(step_ms)))
    value = args.steps / (max_ms * 1e-3)
    # e2e: a fresh partitioned session (network + cold-start state upload,
    # NCCL communicator) running W+K iterations, host wall clock, max over ranks
    n_e2e = args.warmup + args.steps
    nccl_id2 = d.bcast(ga.nccl_unique_id() if d.rank == 0 else None)
    d.barrier()
    t0 = time.perf_counter()
    s2 = ga.Session.distributed(net, cfg, d.rank, d.world, nccl_id2)
    rec2, _ = s2.iterate(n_e2e)
    t_e2e = d.max(time.perf_counter() - t0)
    dims = (net.num_buses, net.num_generators, net.num_branches)
    if d.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": d.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": dict(workload_config(args, dims),
                           parallelism=f"bus-graph partition over {d.world} GPUs, NCCL boundary "
                                       f"exchange"),
            "roofline": {"bound": "fp64", "achieved": None, "peak": None, "unit": "TFLOP/s",
                         "frac": None, "traffic": None,
                         "note": "per-kernel roofline is measured in the N=1 run"},
            "e2e": {"value": len(rec2) / t_e2e, "unit": "iters/s", "wall_s": t_e2e,
                    "iterations": int(len(rec2)), "h2d_bytes_per_step": None,
                    "d2h_bytes_per_step": 56,
                    "note": "gridadmm_session_new_dist (upload, NCCL init) + iterate, max over ranks"},
            "cpu_baseline": None,
            "gpu_launches": 5 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def run_converge(ga, net, dev):
    """Full cold start through gridadmm_solve (driver.cpp:140-246 stop rules),
    preset penalties, default eps 1e-4 / 20 x 1000 iterations; wall clock of
    the call; the reference's quality metrics of the returned solution."""
    cfg = ga.Config(WORKLOAD["preset"], device=dev)
    t0 = time.perf_counter()
    st, rep = ga.solve(net, cfg)
    wall = time.perf_counter() - t0
    m = rep.metrics()
    rep.close()
    out = {"time_to_converge_s": wall, "status": ga.STATUS[st],
           "inner_iterations": int(m["inner_iterations"]),
           "outer_iterations": int(m["outer_iterations"]),
           "iters_per_s": m["inner_iterations"] / wall, "c_inf": m["c_inf"],
           "balance_inf": m["balance_inf"], "limit_violation": m["limit_violation"],
           "bound_violation": m["bound_violation"], "objective": m["objective"],
           "eps": cfg["eps"], "rho": [cfg["rho_pq"], cfg["rho_va"]],
           "note": "gridadmm_solve on a loaded network, wall clock incl. device setup"}
    ref = _load_json(CPU_FULL_SOLVE_FILE)
    if ref:
        out["cpu_full_solve_s"] = ref.get("cpu_time_s")
        out["cpu_full_solve_cores"] = ref.get("cpu_cores")
        out["cpu_full_solve_iterations"] = ref.get("cpu_inner")
        out["cpu_full_solve_source"] = os.path.relpath(CPU_FULL_SOLVE_FILE, REPO)
        out["cpu_objective_bit_identical"] = (
            ref.get("cpu_objective_hex") == float(m["objective"]).hex())
        if ref.get("cpu_time_s"):
            out["speedup_vs_cpu_full_solve"] = ref["cpu_time_s"] / wall
    return out


def run_track(ga, dev):
    """Warm-start tracking, BASELINE configs[4]: ACTIVSg25k-shaped grid,
    30 snapshots (gridcases.synth.ensure_profile), ramp_frac 0.02, preset
    case_ACTIVSg25k; seconds per warm snapshot through gridadmm_track_run."""
    from gridcases import synth
    path = synth.ensure_case("case_ACTIVSg25k", "/tmp/gridadmm_cases")
    net = ga.Network(path)
    prof = synth.ensure_profile(path, periods=30)
    cfg = ga.Config("case_ACTIVSg25k", device=dev, ramp_frac=0.02)
    t0 = time.perf_counter()
    st, trk = ga.track(net, cfg, prof)
    wall = time.perf_counter() - t0
    per = trk.period_table()
    trk.close()
    warm = [p["time_s"] for p in per[1:]]
    out = {"workload": "case_ACTIVSg25k-shaped, 30 snapshots: per-bus multipliers "
                       "P(t)(1+eps), P(t) 1-minute interpolation of an hourly series "
                       "(<=5% swing), eps~N(0,0.005^2); ramp_frac 0.02; gridadmm_track_run",
           "status": ga.STATUS[st], "periods": len(per), "wall_s": wall,
           "cold_s": per[0]["time_s"] if per else None,
           "warm_s_per_step_mean": float(np.mean(warm)) if warm else None,
           "warm_s_per_step_max": float(np.max(warm)) if warm else None,
           "warm_inner_mean": float(np.mean([p["inner"] for p in per[1:]])) if warm else None,
           "c_inf_max": float(max(p["c_inf"] for p in per)) if per else None}
    ref = _load_json(TRACK_CPU_FILE)
    if ref:
        k = int(ref.get("cpu_periods") or 0)
        cpu_mean = ref.get("cpu_warm_s_per_step_mean")
        out["cpu_warm_s_per_step_mean"] = cpu_mean
        out["cpu_periods"] = k
        out["cpu_cores"] = ref.get("cpu_cores")
        out["cpu_source"] = os.path.relpath(TRACK_CPU_FILE, REPO)
        out["cpu_objectives_bit_identical"] = ref.get("objectives_bit_identical")
        if k > 1 and cpu_mean and len(warm) >= k - 1:
            gm = float(np.mean(warm[:k - 1]))  # the same warm snapshots the CPU ran
            out["gpu_warm_s_per_step_mean_same_periods"] = gm
            out["warm_speedup_vs_cpu_same_periods"] = cpu_mean / gm
    return out


def run_b200(args, d: Dist):
    import paper_2110_06879_b200 as ga
    path = case_file(d)
    dev = d.local
    net = ga.Network(path)
    if d.world > 1 or os.environ.get("GRIDADMM_BENCH_DIST") == "1":
        return run_b200_partitioned(args, d, ga, net)
    cfg = ga.Config(WORKLOAD["preset"], device=dev)
    global SOLO
    SOLO = cfg["tile_budget"] > 0  # the solo kernel launches only with a tile budget
    nb, ng, nl, m = net.num_buses, net.num_generators, net.num_branches, net.num_rows

    # --- device-resident timed region -----------------------------------
    sess = ga.Session(net, cfg)
    sess.timed_steps(args.warmup, 0)  # warm-up iterations (untimed)
    k0 = [sess.kernel_time(c) for c in range(6)]
    it0 = sess.step_counters()
    d.barrier()
    with ClockSampler(dev) as clk:
        step_ms, rec = sess.timed_steps(args.steps, L2_FLUSH_BYTES)
    d.barrier()
    k1 = [sess.kernel_time(c) for c in range(6)]
    it1 = sess.step_counters()
    sess.close()
    max_ms = d.max(float(np.sum(step_ms)))
    value = args.steps / (max_ms * 1e-3)

    kern = {name: {"ms_total": k1[c][0] - k0[c][0], "launches": k1[c][1] - k0[c][1]}
            for c, name in enumerate(["generators", "branches", "buses", "zy", "branch_lane_phase",
                                      "branch_tile_solo_phases"])}
    # the generator projection and z / y / residual norms are fused into the
    # bus kernel (kernels.cu bus_block_kernel<true>)
    kern.pop("zy")
    kern.pop("generators")
    # reference-accounted TRON iterations vs trust-region steps the device
    # executed (exact fixed points are skipped, tron.cuh); the roofline counts
    # executed work only
    tron4, tron6 = it1[0] - it0[0], it1[1] - it0[1]
    exec4, exec6 = it1[2] - it0[2], it1[3] - it0[3]
    branch_ms = kern["branches"]["ms_total"]
    census = _load_json(CENSUS_FILE) or {}
    per4 = census.get("per_iter4", CENSUS_FLOPS[4])
    per6 = census.get("per_iter6", CENSUS_FLOPS[6])
    flops = exec4 * per4 + exec6 * per6
    ref_flops = tron4 * per4 + tron6 * per6
    fp64_mul_add, fp64_fma = ga.fp64_peak(dev)
    achieved = flops / (branch_ms * 1e-3) / 1e12 if branch_ms > 0 else 0.0
    # HBM-bound kernels: algorithmic bytes per iteration
    # (with the bus kernel split, "buses" ms is the sum of both launches'
    # durations; the side-stream one shares the SMs with the tile phase)
    hbm_bytes = {"buses": 76 * m + 76 * nb + 64 * ng}
    peaks = _load_json(os.path.join(REPO, "MEASURED_PEAKS.json")) or {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm = {}
    for name, b in hbm_bytes.items():
        t = kern[name]["ms_total"] / max(1, kern[name]["launches"])
        gbs = b / (t * 1e-3) / 1e9 if t > 0 else None
        hbm[name] = {"achieved_gbs": gbs, "bytes": b, "ms": t, "peak_gbs": hbm_peak,
                     "frac": gbs / hbm_peak if gbs else None}
    # DRAM traffic per launch of the dominant kernel and the executed FP64
    # instruction counts, from the committed ncu capture of this workload
    traffic, traffic_note, ncu_fp64 = None, None, None
    try:
        for ln in open(NCU_TRAFFIC_FILE):
            t = json.loads(ln)
            if t.get("kernel") == "lane_kernel" and "dram_bytes" in t:
                traffic = t["dram_bytes"]
                traffic_note = ("lane_kernel dram__bytes_read+write per launch, ncu --set full, "
                                + os.path.relpath(NCU_TRAFFIC_FILE, REPO))
            if t.get("kernel") == "branch_phase_fp64":
                ncu_fp64 = t
    except Exception:  # noqa: BLE001
        pass

    # --- e2e through the C ABI (host buffers) -----------------------------
    e2e = None
    if not args.no_e2e:
        n_e2e = max(args.warmup + args.steps, 200)  # amortizes device setup like a real solve
        cfg2 = ga.Config(WORKLOAD["preset"], device=dev, max_outer=1, max_inner=n_e2e)
        net2 = ga.Network(path)  # host parse (file I/O) outside, like the reference's elapsed_s
        # two back-to-back solves, the second timed: the first one pays the
        # process's one-time costs (lazy module loading of the graph-path
        # kernels, the device pool's growth); each solve still allocates,
        # uploads, captures its graph and downloads inside the timed region
        for rep_i in range(2):
            d.barrier()
            t0 = time.perf_counter()
            st, rep = ga.solve(net2, cfg2)  # network H2D, cold start, iterations, solution D2H
            pg, qg = rep.dispatch()
            vm, va = rep.voltages()
            t_e2e = time.perf_counter() - t0
            n_it = rep.metric("inner_iterations")
            rep.close()
        net2.close()
        t_max = d.max(t_e2e)
        h2d = (8 * (6 * ng + 10 * nl + 6 * nb) + 4 * (3 * nl + 7 * nb + m))  # network SoA
        d2h = 56 * n_it + 8 * (2 * ng + 2 * nb)
        e2e = {"value": n_it / t_max, "unit": "iters/s",
               "h2d_bytes_per_step": h2d / n_it, "d2h_bytes_per_step": d2h / n_it,
               "wall_s": t_max, "iterations": int(n_it),
               "note": "gridadmm_solve(max_outer=1, max_inner=max(W+K, 200)) on a loaded network + "
                       "dispatch/voltages: device alloc, network upload, device cold start, "
                       "graph capture, the loop's record readbacks, solution download (file parse "
                       "excluded); the second of two back-to-back solves"}

    # --- CPU baseline (reference on host cores), rank 0 only ---------------
    cpu = None
    if d.rank == 0 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        ksteps = min(args.cpu_steps, args.steps)
        try:
            rate, dt, wall, series, _ = reference_run(path, args.warmup, ksteps, workers)
            same = bool(np.array_equal(
                series[args.warmup:args.warmup + ksteps, 2:5].view(np.uint64),
                rec[:ksteps, 0:3].view(np.uint64)))
            cpu = {"value": rate, "unit": "iters/s", "cores": workers, "kind": "reference",
                   "sample": f"inner iterations {args.warmup}..{args.warmup + ksteps - 1} of the "
                             f"same cold start ({dt:.1f} s of {wall:.1f} s wall), reference C++ "
                             f"solver (oracle/_ref) via its C ABI, workers={workers}",
                   "residuals_bit_identical_to_gpu": same}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "iters/s", "cores": workers, "kind": "reference",
                   "sample": f"failed: {e}"}

    conv = None
    if d.rank == 0 and not args.no_converge:
        try:
            conv = run_converge(ga, net, dev)
        except Exception as e:  # noqa: BLE001
            conv = {"failed": str(e)}
    track = None
    if d.rank == 0 and not args.no_track:
        try:
            track = run_track(ga, dev)
        except Exception as e:  # noqa: BLE001
            track = {"failed": str(e)}

    if d.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": d.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": workload_config(args, (nb, ng, nl)),
            "roofline": {"bound": "fp64",
                         "kernel": "branch phase: lane_kernel + tile_kernel + solo_kernel (TRON NLPs)",
                         "achieved": achieved, "peak": fp64_mul_add, "unit": "TFLOP/s",
                         "frac": achieved / fp64_mul_add if fp64_mul_add else None,
                         "traffic": traffic, "traffic_note": traffic_note,
                         "peak_note": "measured DMUL+DADD issue rate on this GPU "
                                      "(gridadmm_probe_fp64_peak; kernels built -fmad=false); "
                                      f"DFMA peak {fp64_fma:.1f} TFLOP/s",
                         "flops_per_launch": flops / max(1, kern["branches"]["launches"]),
                         "census_flops_per_tron_iteration": {"n4": per4, "n6": per6,
                                                             "source": census.get("source")},
                         "tron_iterations_reference": [tron4, tron6],
                         "tron_steps_executed": [exec4, exec6],
                         "ncu_executed_fp64": ncu_fp64,
                         "reference_equivalent_tflops": (ref_flops / (branch_ms * 1e-3) / 1e12
                                                         if branch_ms > 0 else None)},
            "roofline_hbm": hbm,
            "kernels": kern,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "converge": conv,
            "track": track,
            "gpu_launches": (3 + (1 if SOLO else 0) + (2 if BUS_OVERLAP else 1)) * args.steps,
            "gpu_launches_note": ("per step: reset_scalars_kernel, lane_kernel, tile_kernel, "
                                  + ("solo_kernel, " if SOLO else "")
                                  + "bus_block_kernel (generator projection, z, y and "
                                  "norms fused in)"
                                  + (" twice: the buses not adjacent to a branch handed to the "
                                     "tile phase on a side stream beside the tile / solo "
                                     "kernels, the rest after them (plus a 70 KB flag memset)"
                                     if BUS_OVERLAP else "")
                                  + "; the L2-flush memset excluded"),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    d = Dist()
    try:
        if args.impl == "reference":
            run_reference_arm(args, d)
        else:
            run_b200(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
