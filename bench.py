#!/usr/bin/env python3
"""bench.py — ADMM iterations/s of the B200-native gridadmm on an
ACTIVSg70k-shaped grid (BASELINE.json metric, config[3]).

A "step" is one inner ADMM iteration of the two-level ADMM (generator
projection -> branch NLPs -> bus consensus -> z/y/residual norms, plus the
host's read of the four residual norms that drive the loop control;
proj/src/driver.cpp:155-186) over the whole grid.  The first W iterations
from the cold start are the warm-up, the next K are timed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

* `value`: K x ranks / max-over-ranks device time of the K steps, state
  resident in HBM, each step timed with CUDA events on the solver's stream
  and an L2 flush (256 MiB write) between steps outside the events.
* `e2e`: the same metric through the public C ABI with host buffers:
  gridadmm_network_load'ed case -> gridadmm_solve (max_outer 1, max_inner
  W+K; network + state upload, every iteration's norm readback and the
  solution download inside the wall-clock region).
* `roofline`: the branch-NLP kernel (dominant) against the measured FP64
  DMUL+DADD peak (the kernel is built with -fmad=false for bit-exactness).
* `cpu_baseline`: the reference C++ solver (oracle/_ref, compiled from the
  reference sources with the pinned sincos) on this host's cores, timing a
  bounded sample of the SAME iterations (its trajectory is bit-identical).
* `converge`: time-to-converge of a full cold-start solve on the device
  (penalty (100, 1e4), see CONVERGE_RHO) and a late-solve window (outer
  iteration 10) timed on the device and with the reference CPU solver from
  the same state (bit-identical residuals checked).
* `--impl reference`: that reference solver alone (rank 0), same metric.

Multi-GPU (torchrun, N>1): the 70k-shaped grid is split over the N GPUs by
the bus-graph partition, NCCL boundary exchange ("scaling": "strong");
DESIGN.md §7.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

L2_FLUSH_BYTES = 256 << 20
SHAPE = "case_ACTIVSg70k"
# Lean FP64 op census per TRON iteration (flops whose results are consumed,
# branch evaluation + TRON core, amortized per-branch setup included),
# measured with the C restatement's counters (oracle/gridadmm_oracle.c FL())
# on the case2868rte-shaped synthetic grid, ACTIVSg70k preset, inner
# iterations 1-20: 4-var 1588, 6-var 3329 flops/iteration.
CENSUS_FLOPS = {4: 1588.0, 6: 3329.0}
# Time-to-converge run: the synthetic ACTIVSg70k-shaped grid is not the real
# case, and the paper's penalty pair for it (3e4 / 3e5) does not converge on
# it in 20 x 1000 iterations; (100, 1e4) — the reference's own choice for its
# bundled cases (proj/tests/acceptance.cpp:58-69) — converges (rho sweep,
# scripts/rho_sweep.py).
CONVERGE_RHO = (100.0, 1e4)
LATE_OUTER = 10   # the late-window sample starts at this outer iteration
LATE_STEPS = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--shape", default=SHAPE)
    ap.add_argument("--seed", type=int, default=2110)
    ap.add_argument("--preset", default="case_ACTIVSg70k")
    ap.add_argument("--cpu-steps", type=int, default=30, help="timed iterations of the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-converge", action="store_true",
                    help="skip the time-to-converge run (full cold-start solve)")
    return ap.parse_args()


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

    def sum(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
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


def case_file(shape: str, seed: int, d: Dist) -> str:
    from paper_2110_06879_b200 import synth
    directory = os.path.join("/tmp", "gridadmm_cases")
    path = os.path.join(directory, f"{shape}_synth_s{seed}.m")
    if d.rank == 0:
        synth.ensure_case(shape, directory, seed=seed)
    d.barrier()
    while not os.path.exists(path):  # ranks on the same host share /tmp
        time.sleep(0.2)
    return path


def cfg_kwargs(args, max_inner):
    return dict(max_outer=1, max_inner=max_inner)


def reference_rate(path, args, iters_timed, workers):
    """Reference C++ solver (oracle/_ref) on host cores: iterations/s over
    iterations W..W+iters_timed-1 from the elapsed_s stamps of its own series
    (proj/src/driver.cpp:190-191)."""
    import oracle
    from paper_2110_06879_b200 import Config
    if not oracle.have_ref():
        raise RuntimeError("oracle/_ref/libgridadmm_ref.so missing")
    c = Config(args.preset)
    ref = oracle.RefNet(path)
    n = args.warmup + iters_timed
    t0 = time.perf_counter()
    series, info, _ = ref.solve(rho_pq=c["rho_pq"], rho_va=c["rho_va"], max_outer=1,
                                max_inner=n, workers=workers)
    wall = time.perf_counter() - t0
    el = series[:, 5]
    start = el[args.warmup - 1] if args.warmup > 0 else 0.0
    dt = el[n - 1] - start
    return iters_timed / dt, dt, wall, series


def run_reference_arm(args, d: Dist):
    if d.rank != 0:
        return
    path = case_file(args.shape, args.seed, d) if d.world == 1 else None
    if path is None:
        from paper_2110_06879_b200 import synth
        path = synth.ensure_case(args.shape, "/tmp/gridadmm_cases", seed=args.seed)
    workers = os.cpu_count() or 1
    rate, dt, wall, _ = reference_rate(path, args, args.steps, workers)
    line = {
        "metric": "ADMM iters/sec & time-to-converge (s) on ACTIVSg70k; warm-start track s/step",
        "impl": "reference", "value": rate, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded tiling of MATPOWER case30/case118 to ACTIVSg70k dims)",
        "config": {"workload": f"{args.shape}-shaped cold start, inner iterations "
                               f"{args.warmup}..{args.warmup + args.steps - 1}",
                   "preset": args.preset, "seed": args.seed},
        "cpu_baseline": {"value": rate, "unit": "iters/s", "cores": workers, "kind": "reference",
                         "sample": f"{args.steps} timed inner iterations after {args.warmup} "
                                   f"warm-up, reference C++ solver, workers={workers}"},
        "e2e": {"value": rate, "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_partitioned(args, d: Dist, ga, path, net):
    """N > 1: one ACTIVSg70k-shaped grid split over N GPUs by the bus-graph
    partition (strong scaling); every step is one ADMM iteration of the whole
    grid, boundary rows and residual norms exchanged with NCCL inside the
    library.  Device time per step from CUDA events on each rank's stream,
    max over ranks."""
    dev = d.local
    cfg = ga.Config(args.preset, device=dev)
    nccl_id = d.bcast(ga.nccl_unique_id() if d.rank == 0 else None)
    sess = ga.Session.distributed(net, cfg, d.rank, d.world, nccl_id)
    sess.timed_steps(args.warmup, 0)
    d.barrier()
    with ClockSampler(dev) as clk:
        step_ms, rec = sess.timed_steps(args.steps, L2_FLUSH_BYTES)
    d.barrier()
    max_ms = d.max(float(np.sum(step_ms)))
    value = args.steps / (max_ms * 1e-3)
    # e2e: open a fresh partitioned session (network + cold-start state upload,
    # NCCL communicator) and run W+K iterations, host wall clock, max over ranks
    n_e2e = max(args.warmup + args.steps, 200)
    nccl_id2 = d.bcast(ga.nccl_unique_id() if d.rank == 0 else None)
    d.barrier()
    t0 = time.perf_counter()
    s2 = ga.Session.distributed(net, cfg, d.rank, d.world, nccl_id2)
    rec2, _ = s2.iterate(n_e2e)
    t_e2e = d.max(time.perf_counter() - t0)
    nb, ng, nl, m = net.num_buses, net.num_generators, net.num_branches, net.num_rows
    conv = None
    if d.rank == 0 and d.world == 1 and not args.no_converge:
        try:
            conv = run_converge(args, ga, net, path, dev)
        except Exception as e:  # noqa: BLE001
            conv = {"failed": str(e)}

    if d.rank == 0:
        line = {
            "metric": "ADMM iters/sec & time-to-converge (s) on ACTIVSg70k; warm-start track s/step",
            "value": value, "unit": "iters/s", "n_gpus": d.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded tiling of MATPOWER case30/case118 to ACTIVSg70k dims)",
            "config": {"workload": f"{args.shape}-shaped ({nb} buses, {ng} gens, {nl} branches, "
                                   f"m={m}) cold start, inner iterations "
                                   f"{args.warmup}..{args.warmup + args.steps - 1}",
                       "preset": args.preset, "seed": args.seed,
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "parallelism": f"bus-graph partition over {d.world} GPUs, NCCL boundary "
                                      f"exchange"},
            "roofline": {"bound": "fp64", "kernel": "branch NLP kernels", "achieved": None,
                         "peak": None, "unit": "TFLOP/s", "frac": None, "traffic": None,
                         "note": "per-kernel roofline is measured in the N=1 run"},
            "e2e": {"value": len(rec2) / t_e2e, "unit": "iters/s", "wall_s": t_e2e,
                    "iterations": int(len(rec2)), "h2d_bytes_per_step": None,
                    "d2h_bytes_per_step": 56,
                    "note": "gridadmm_session_new_dist (upload, NCCL init) + iterate, max over ranks"},
            "cpu_baseline": None,
            "gpu_launches": 10 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def run_converge(args, ga, net, path, dev):
    """Time-to-converge of a cold start (eps 1e-4, 20 x 1000 iterations) on
    the device, driven exactly like driver.cpp:152-239 (inner loops with the
    reference's stop tests inside gridadmm_session_iterate, outer updates
    with the beta schedule), wall clock from session creation.  At the start
    of outer iteration LATE_OUTER the full state is snapshotted (excluded
    from the wall time); from it the reference C++ solver (all host cores)
    and a fresh device session each run LATE_STEPS iterations: the late-solve
    rate of both, with bit-identical residual series."""
    import oracle
    eps, max_inner, max_outer = 1e-4, 1000, 20
    cfg = ga.Config(rho_pq=CONVERGE_RHO[0], rho_va=CONVERGE_RHO[1], eps=eps, device=dev,
                    max_inner=max_inner, max_outer=max_outer)
    t0 = time.perf_counter()
    paused = 0.0
    s = ga.Session(net, cfg)
    prev, status, iters, snap, outer = -1.0, "ERR_ITERATION_LIMIT", 0, None, 0
    for outer in range(1, max_outer + 1):
        if outer == LATE_OUTER:
            tp = time.perf_counter()
            snap = (s.get_state(), iters)
            paused += time.perf_counter() - tp
        rec, why = s.iterate(max_inner)
        iters += len(rec)
        if why == 2:
            status = "ERR_DIVERGED"
            break
        z = float(rec[-1, 2])
        if z <= eps:
            status = "OK"
            break
        s.phase("outer", z, prev)
        prev = z
    wall = time.perf_counter() - t0 - paused
    s.close()
    out = {"time_to_converge_s": wall, "status": status, "inner_iterations": iters,
           "outer_iterations": outer, "iters_per_s": iters / wall,
           "rho": list(CONVERGE_RHO), "eps": eps,
           "note": "device session driven with driver.cpp's loop control; wall clock incl. setup"}
    if snap is not None and oracle.have_ref():
        st, at = snap
        s2 = ga.Session(net, cfg)
        s2.set_state(st)
        ms, rec = s2.timed_steps(LATE_STEPS, L2_FLUSH_BYTES)
        s2.close()
        workers = os.cpu_count() or 1
        ref = oracle.RefNet(path)
        series, _, _ = ref.solve(init=st, rho_pq=CONVERGE_RHO[0], rho_va=CONVERGE_RHO[1], eps=eps,
                                 max_outer=1, max_inner=LATE_STEPS, workers=workers)
        el = series[:, 5]
        gpu_rate = LATE_STEPS / (float(np.sum(ms)) * 1e-3)
        cpu_rate = LATE_STEPS / float(el[-1]) if el[-1] > 0 else None
        out["late_window"] = {
            "start_iteration": at, "beta": float(st["beta"][0]), "steps": LATE_STEPS,
            "gpu_iters_per_s": gpu_rate, "cpu_iters_per_s": cpu_rate, "cpu_cores": workers,
            "gpu_over_cpu": gpu_rate / cpu_rate if cpu_rate else None,
            "residuals_bit_identical": bool(np.array_equal(
                series[:LATE_STEPS, 2:5].view(np.uint64), rec[:LATE_STEPS, 0:3].view(np.uint64)))}
    return out


def run_b200(args, d: Dist):
    import paper_2110_06879_b200 as ga
    path = case_file(args.shape, args.seed, d)
    dev = d.local
    net = ga.Network(path)
    cfg = ga.Config(args.preset, device=dev)
    nb, ng, nl, m = net.num_buses, net.num_generators, net.num_branches, net.num_rows

    if d.world > 1 or os.environ.get("GRIDADMM_BENCH_DIST") == "1":
        return run_b200_partitioned(args, d, ga, path, net)

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
    my_ms = float(np.sum(step_ms))
    max_ms = d.max(my_ms)
    total_iters = d.sum(float(args.steps))
    value = total_iters / (max_ms * 1e-3)

    kern = {name: {"ms_total": k1[c][0] - k0[c][0], "launches": k1[c][1] - k0[c][1]}
            for c, name in enumerate(["generators", "branches", "buses", "zy", "branch_lane_phase",
                                      "branch_tile_solo_phases"])}
    kern.pop("zy")  # z / y / residual norms are fused into the bus kernel
    # reference-accounted TRON iterations vs trust-region steps the device
    # executed (exact fixed points are skipped, tron.cuh); the roofline counts
    # executed work only
    tron4, tron6 = it1[0] - it0[0], it1[1] - it0[1]
    exec4, exec6 = it1[2] - it0[2], it1[3] - it0[3]
    branch_ms = kern["branches"]["ms_total"]
    flops = exec4 * CENSUS_FLOPS[4] + exec6 * CENSUS_FLOPS[6]
    ref_flops = tron4 * CENSUS_FLOPS[4] + tron6 * CENSUS_FLOPS[6]
    fp64_mul_add, fp64_fma = ga.fp64_peak(dev)
    achieved = flops / (branch_ms * 1e-3) / 1e12 if branch_ms > 0 else 0.0
    # HBM-bound phases: algorithmic bytes per iteration
    # generators: 4 row arrays x 2 rows + 6 params read, 2 rows written;
    # buses (fused with z / y / norms): per row the CSR index + rho, x, z, y,
    # xbar, lambda read and xbar, z, y written (76 B), per bus 7 CSR offsets
    # + gs, bs, pd, qd read and w, theta written (76 B)
    hbm_bytes = {"generators": 128 * ng, "buses": 76 * m + 76 * nb}
    hbm = {}
    for name, b in hbm_bytes.items():
        t = kern[name]["ms_total"] / max(1, kern[name]["launches"])
        hbm[name] = {"gbs": b / (t * 1e-3) / 1e9 if t > 0 else None, "bytes": b, "ms": t}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # DRAM traffic per launch of the dominant kernel from the committed ncu
    # --set full capture (profiles/r01_ncu_traffic.jsonl, inner iteration 10)
    traffic, traffic_note = None, None
    try:
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for ln in open(os.path.join(REPO, "profiles", "r01_ncu_traffic.jsonl")):
            t = json.loads(ln)
            if t["kernel"] == "lane_kernel":
                traffic = t["dram_read"][0] * unit[t["dram_read"][1]] + \
                    t["dram_write"][0] * unit[t["dram_write"][1]]
                traffic_note = ("lane_kernel dram__bytes_read+write per launch, ncu --set full, "
                                "profiles/r01_ncu_traffic.jsonl; the phase is FP64-latency bound")
    except Exception:  # noqa: BLE001
        pass

    # --- e2e through the C ABI (host buffers) -----------------------------
    e2e = None
    if not args.no_e2e:
        n_e2e = max(args.warmup + args.steps, 200)
        cfg2 = ga.Config(args.preset, device=dev, max_outer=1, max_inner=n_e2e)
        net2 = ga.Network(path)  # host parse (file I/O) outside, like the reference's elapsed_s
        d.barrier()
        t0 = time.perf_counter()
        st, rep = ga.solve(net2, cfg2)  # network + state H2D, iterations, solution D2H
        pg, qg = rep.dispatch()
        vm, va = rep.voltages()
        t_e2e = time.perf_counter() - t0
        n_it = rep.metric("inner_iterations")
        t_max = d.max(t_e2e)
        h2d = (8 * (6 * ng + 10 * nl + 6 * nb) + 4 * (3 * nl + 7 * nb + m)  # network
               + 8 * (6 * m + 2 * nb + 9 * nl))  # cold-start state
        d2h = 56 * n_it + 8 * (2 * ng + 2 * nb)
        e2e = {"value": d.sum(n_it) / t_max, "unit": "iters/s",
               "h2d_bytes_per_step": h2d / n_it, "d2h_bytes_per_step": d2h / n_it,
               "wall_s": t_max, "iterations": int(n_it),
               "note": "gridadmm_solve(max_outer=1) on a loaded network + dispatch/voltages: "
                       "device alloc, network+state upload, cold start, every iteration's "
                       "norm readback, solution download (file parse excluded)"}

    # --- CPU baseline (reference on host cores), rank 0 only ---------------
    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        ksteps = min(args.cpu_steps, args.steps)
        try:
            rate, dt, wall, series = reference_rate(path, args, ksteps, workers)
            # same trajectory: the reference's residuals must equal ours bit-for-bit
            same = bool(np.array_equal(series[args.warmup:args.warmup + ksteps, 2:5].view(np.uint64),
                                       rec[:ksteps, 0:3].view(np.uint64)))
            cpu = {"value": rate, "unit": "iters/s", "cores": workers, "kind": "reference",
                   "sample": f"inner iterations {args.warmup}..{args.warmup + ksteps - 1} of the "
                             f"same cold start ({dt:.1f} s of {wall:.1f} s wall), reference C++ "
                             f"solver from oracle/_ref, workers={workers}",
                   "residuals_bit_identical_to_gpu": same}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "iters/s", "cores": workers, "kind": "reference",
                   "sample": f"failed: {e}"}

    conv = None
    if d.rank == 0 and d.world == 1 and not args.no_converge:
        try:
            conv = run_converge(args, ga, net, path, dev)
        except Exception as e:  # noqa: BLE001
            conv = {"failed": str(e)}

    if d.rank == 0:
        line = {
            "metric": "ADMM iters/sec & time-to-converge (s) on ACTIVSg70k; warm-start track s/step",
            "value": value, "unit": "iters/s", "n_gpus": d.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded tiling of MATPOWER case30/case118 to ACTIVSg70k dims)",
            "config": {"workload": f"{args.shape}-shaped ({nb} buses, {ng} gens, {nl} branches, "
                                   f"m={m}) cold start, inner iterations "
                                   f"{args.warmup}..{args.warmup + args.steps - 1}",
                       "preset": args.preset, "seed": args.seed,
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "parallelism": "replicas" if d.world > 1 else "single GPU"},
            "roofline": {"bound": "fp64",
                         "kernel": "branch phase: lane_kernel + tile_kernel + solo_kernel (TRON NLPs)",
                         "achieved": achieved, "peak": fp64_mul_add, "unit": "TFLOP/s",
                         "frac": achieved / fp64_mul_add if fp64_mul_add else None,
                         "traffic": traffic, "traffic_note": traffic_note,
                         "peak_note": "measured DMUL+DADD issue rate (kernel built -fmad=false); "
                                      f"DFMA peak {fp64_fma:.1f} TFLOP/s",
                         "flops_per_launch": flops / max(1, kern["branches"]["launches"]),
                         "tron_iterations_reference": [tron4, tron6],
                         "tron_steps_executed": [exec4, exec6],
                         "reference_equivalent_tflops": (ref_flops / (branch_ms * 1e-3) / 1e12
                                                         if branch_ms > 0 else None)},
            "roofline_hbm": {k: dict(v, peak_gbs=hbm_peak,
                                     frac=(v["gbs"] / hbm_peak if v["gbs"] else None))
                             for k, v in hbm.items()},
            "kernels": kern,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "converge": conv,
            "gpu_launches": 6 * args.steps,
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
