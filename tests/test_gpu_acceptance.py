"""The reference's end-to-end acceptance criteria (proj/tests/acceptance.cpp)
and failure semantics, on the sm_100a path, each checked against the
reference solver run on the same input:

* criterion 4 — desk-scale cold starts (case30, case118) through
  gridadmm_solve: status, iteration counts, every report metric bit for bit,
  convergence.csv bit for bit, solution.json byte for byte (wall-clock
  phase_times_s excepted), plus the criterion's own bars;
* criterion 6 — case30 10-period tracking: per-period counts / metrics bit
  for bit, periods.csv byte for byte (time_s excepted), ramp windows held;
* criterion 8 — warm restart from the converged case9 state;
* failure paths: NumericalError -> restore the previous point
  (kernels.cpp:273-274), DIVERGED early return (driver.cpp:193-204),
  SingularBusError -> GRIDADMM_ERR_INTERNAL (kernels.cpp:408-412).
"""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import case_path

pytestmark = pytest.mark.gpu

DESK = {  # proj/tests/acceptance.cpp:58-69
    "case9": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5, max_inner=1000),
    "case30": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5, max_inner=1000),
    "case118": dict(rho_pq=100.0, rho_va=1e4, eps=1e-6, max_inner=300),
}
FIELDS = ("x", "xbar", "z", "y", "lambda", "rho", "bus_w", "bus_theta", "branch_point", "lt_ij",
          "lt_ji", "rho_tilde", "beta")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_state_equal(a, b, where):
    for f in FIELDS:
        if not np.array_equal(bits(a[f]), bits(b[f])):
            k = np.nonzero(bits(a[f]) != bits(b[f]))[0][0]
            raise AssertionError(f"{where}: {f}[{k}] {a[f].ravel()[k]!r} vs {b[f].ravel()[k]!r}")


class RefCapi:
    """The reference library through its own C ABI (oracle/_ref)."""

    def __init__(self, oracle_mod, path, **cfg):
        self.h = h = oracle_mod.ref_capi()
        self.net = ctypes.c_void_p()
        assert h.gridadmm_network_load(os.fsencode(path), ctypes.byref(self.net)) == 0
        self.cfg = h.gridadmm_config_new()
        for k, v in cfg.items():
            assert h.gridadmm_config_set(self.cfg, k.encode(), float(v)) == 0, k
        self.metrics = oracle_mod.ref_metrics

    def solve(self):
        rep = ctypes.c_void_p()
        st = self.h.gridadmm_solve(self.net, self.cfg, ctypes.byref(rep))
        return st, rep

    def close(self):
        self.h.gridadmm_config_free(self.cfg)
        self.h.gridadmm_network_free(self.net)


def mask_wall_clock_json(text):
    return re.sub(r'("phase_times_s": \{)[^}]*(\})', r"\1\2", text)


def csv_drop_column(text, name):
    rows = [ln.split(",") for ln in text.strip("\n").split("\n")]
    k = rows[0].index(name)
    return "\n".join(",".join(r[:k] + r[k + 1:]) for r in rows)


@pytest.mark.parametrize("name", ["case30", "case118"])
def test_desk_cold_start_matches_reference(gridadmm, oracle_mod, tmp_path, name):
    d = DESK[name]
    net = gridadmm.Network(case_path(name))
    cfg = gridadmm.Config(**d)
    st, rep = gridadmm.solve(net, cfg)
    ref = RefCapi(oracle_mod, case_path(name), **d)
    rst, rrep = ref.solve()
    assert st == rst == 0
    m, rm = rep.metrics(), ref.metrics(ref.h, rrep)
    for k in rm:
        assert bits(m[k]) == bits(rm[k]), (k, m[k], rm[k])
    # the criterion's own bars (acceptance.cpp:544-549); the reference meets them too
    conv = tmp_path / "conv.csv"
    rep.write_convergence(str(conv))
    rows = np.loadtxt(conv, delimiter=",", skiprows=1, ndmin=2)
    assert rows[-1, 4] <= 1e-4 and m["c_inf"] <= 1e-3
    # convergence.csv: every column but elapsed_s, byte for byte
    rconv = tmp_path / "rconv.csv"
    assert ref.h.gridadmm_report_write_convergence(rrep, os.fsencode(str(rconv))) == 0
    assert csv_drop_column(conv.read_text(), "elapsed_s") == \
        csv_drop_column(rconv.read_text(), "elapsed_s")
    # solution.json with a reference objective (gap key), byte for byte
    sol, rsol = tmp_path / "s.json", tmp_path / "rs.json"
    rep.write_solution(str(sol), 5000.0)
    assert ref.h.gridadmm_report_write_solution(rrep, os.fsencode(str(rsol)), 5000.0) == 0
    assert mask_wall_clock_json(sol.read_text()) == mask_wall_clock_json(rsol.read_text())
    # dispatch / voltages getters
    pg, qg = rep.dispatch()
    rpg, rqg = np.zeros_like(pg), np.zeros_like(qg)
    ref.h.gridadmm_report_dispatch(rrep, rpg.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   rqg.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert np.array_equal(bits(pg), bits(rpg)) and np.array_equal(bits(qg), bits(rqg))
    ref.h.gridadmm_report_free(rrep)
    ref.close()


def test_tracking_case30_ten_periods(gridadmm, oracle_mod, tmp_path):
    """acceptance.cpp:627-684 (criterion 6) through gridadmm_track_run."""
    mult = [1.0, 1.005, 1.010, 1.015, 1.020, 1.015, 1.010, 1.005, 1.0, 0.995]
    csv = tmp_path / "p.csv"
    csv.write_text("period,multiplier\n" + "".join(f"{t + 1},{v}\n" for t, v in enumerate(mult)))
    d = dict(DESK["case30"], ramp_frac=0.02)
    net = gridadmm.Network(case_path("case30"))
    st, trk = gridadmm.track(net, gridadmm.Config(**d), str(csv))
    rst, ref = oracle_mod.ref_track(case_path("case30"), str(csv), "case30",
                                    **{k: v for k, v in d.items() if k not in ("rho_pq", "rho_va")})
    assert st == rst == 0
    assert trk.num_periods == len(ref) == 10
    prev = None
    pmax = net.export()["gen"][:, 2]  # (bus, pmin, pmax, ...)
    warm = 0
    for p, rm in enumerate(ref, start=1):
        r = trk.period_report(p)
        m = r.metrics()
        for k in ("objective", "c_inf", "balance_inf", "limit_violation", "bound_violation",
                  "inner_iterations", "outer_iterations", "branch_solve_failures"):
            assert bits(m[k]) == bits(rm[k]), (p, k)
        pg, _ = r.dispatch()
        if prev is not None:
            warm += m["inner_iterations"]
            assert np.max(np.abs(pg - prev) - 0.02 * pmax) <= 1e-8  # acceptance.cpp:656-662
        prev = pg
    cold = trk.period_report(1).metric("inner_iterations")
    assert warm < 4.5 * cold  # acceptance.cpp:668-670
    # periods.csv with reference objectives: byte for byte but time_s
    refs = [float(rm["objective"]) * 1.001 for rm in ref]
    out = tmp_path / "periods.csv"
    trk.write_periods(str(out), refs)
    h = oracle_mod.ref_capi()
    rnet = ctypes.c_void_p()
    assert h.gridadmm_network_load(os.fsencode(case_path("case30")), ctypes.byref(rnet)) == 0
    c = h.gridadmm_config_new()
    assert h.gridadmm_config_preset(c, b"case30") == 0
    for k, v in d.items():
        assert h.gridadmm_config_set(c, k.encode(), float(v)) == 0
    rtrk = ctypes.c_void_p()
    assert h.gridadmm_track_run(rnet, c, os.fsencode(str(csv)), ctypes.byref(rtrk)) == 0
    rout = tmp_path / "rperiods.csv"
    arr = (ctypes.c_double * len(refs))(*refs)
    assert h.gridadmm_track_write_periods(rtrk, os.fsencode(str(rout)), arr, len(refs)) == 0
    assert csv_drop_column(out.read_text(), "time_s") == csv_drop_column(rout.read_text(), "time_s")
    h.gridadmm_track_free(rtrk)
    h.gridadmm_config_free(c)
    h.gridadmm_network_free(rnet)


def test_fixed_point_warm_restart(gridadmm, oracle_mod):
    """acceptance.cpp:688-703 (criterion 8): a solve started from the
    converged case9 state stops after one outer / <= 2 inner iterations, with
    the reference's exact counts, metrics and final state."""
    d = DESK["case9"]
    net = gridadmm.Network(case_path("case9"))
    cfg = gridadmm.Config(**d)
    sess = gridadmm.Session(net, cfg)
    st1, rep1 = sess.solve(cfg, warm=False)
    st2, rep2 = sess.solve(cfg, warm=True)
    ref = oracle_mod.RefNet(case_path("case9"))
    _, info1, fin1 = ref.solve(**d)
    _, info2, fin2 = ref.solve(init=fin1, **d)
    assert st1 == st2 == 0 and info1[0] == info2[0] == 0
    m2 = rep2.metrics()
    assert m2["outer_iterations"] == info2[1] == 1
    assert m2["inner_iterations"] == info2[2] <= 2
    assert bits(m2["objective"]) == bits(info2[4])
    assert_state_equal(sess.get_state(), fin2, "after the warm restart")


def test_numerical_error_restores_previous_point(gridadmm, oracle_mod):
    """A branch whose objective is not finite at the start point fails its
    TRON solve: the previous point is kept, its consensus rows are rewritten
    from it, and the failure is counted (kernels.cpp:246-281)."""
    d = DESK["case30"]
    net = gridadmm.Network(case_path("case30"))
    sess = gridadmm.Session(net, gridadmm.Config(**d))
    ref = oracle_mod.RefNet(case_path("case30"))
    s = ref.cold_start(**d)
    for _ in range(3):
        for p in ("generators", "branches", "buses", "z", "y"):
            ref.phase(gridadmm.PHASES[p], s, **d)
    ng = net.num_generators
    bad = [0, 5, 17]  # one limited and some unlimited branches
    for b in bad:
        s["y"][2 * ng + 8 * b] = np.inf
    s["y"][2 * ng + 8 * 40 + 4] = np.nan
    sess.set_state(s)
    fails = sess.phase("branches")
    rfails = ref.phase(gridadmm.PHASES["branches"], s, **d)
    assert fails == rfails >= len(bad) + 1
    assert_state_equal(sess.get_state(), s, "branch phase with non-finite data")


def test_diverged_early_return(gridadmm, oracle_mod):
    """Residuals past 1e8 end the solve with DIVERGED and a report
    (driver.cpp:193-204; gridadmm.h:62)."""
    d = DESK["case9"]
    net = gridadmm.Network(case_path("case9"))
    cfg = gridadmm.Config(**d)
    ref = oracle_mod.RefNet(case_path("case9"))
    for field, value in (("y", 1e6), ("lambda", 1e7)):  # diverge at inner 1 / inner 2
        s = ref.cold_start(**d)
        s[field][:] = value
        sess = gridadmm.Session(net, cfg)
        sess.set_state(s)
        st, rep = sess.solve(cfg, warm=True)
        series, info, fin = ref.solve(init=s, **d)
        assert info[0] == 2 and st == 5  # SolveStatus::Diverged -> GRIDADMM_ERR_DIVERGED
        m = rep.metrics()
        assert m["inner_iterations"] == info[2] and m["outer_iterations"] == info[1]
        assert bits(m["objective"]) == bits(info[4])
        assert_state_equal(sess.get_state(), fin, f"diverged, {field}={value}")


def test_singular_bus_is_internal_error(gridadmm, oracle_mod, tmp_path):
    """An isolated bus makes its balance system singular: SingularBusError in
    the bus phase (kernels.cpp:364-391,408-412), GRIDADMM_ERR_INTERNAL at the
    ABI, with the reference's bus index in the phase replay."""
    txt = open(case_path("case9")).read()
    row9 = "\t9\t1\t125\t50\t0\t0\t1\t1\t0\t345\t1\t1.1\t0.9;\n"
    assert row9 in txt
    path = tmp_path / "case9_isolated.m"
    path.write_text(txt.replace(row9, row9 + "\t10\t1\t0\t0\t0\t0\t1\t1\t0\t345\t1\t1.1\t0.9;\n"))
    d = DESK["case9"]
    net = gridadmm.Network(str(path))
    with pytest.raises(gridadmm.GridAdmmError) as e:
        gridadmm.solve(net, gridadmm.Config(**d))
    ref = RefCapi(oracle_mod, str(path), **d)
    rst, rrep = ref.solve()
    ref.close()
    assert e.value.status == rst == 7 and not rrep.value
    assert "10" in e.value.message
    sess = gridadmm.Session(net, gridadmm.Config(**d))
    rnet = oracle_mod.RefNet(str(path))
    s = rnet.cold_start(**d)
    for p in ("generators", "branches"):
        rnet.phase(gridadmm.PHASES[p], s, **d)
    sess.set_state(s)
    got = sess.phase("buses")
    want = rnet.phase(gridadmm.PHASES["buses"], s, **d)
    assert got == want == 9


@pytest.mark.parametrize("max_inner", [20, 200])
def test_device_metrics_with_line_limit_violation(gridadmm, oracle_mod, tmp_path, max_inner):
    """Device extraction + metrics (extract.cu; driver.cpp:65-138) on a
    solution that violates a line limit, so the glibc-hypot candidate path is
    exercised: every metric bit, dispatch, voltages and solution.json."""
    txt = open(case_path("case9")).read()
    row = "\t5\t6\t0.039\t0.17\t0.358\t150\t150\t150\t0\t0\t1\t-360\t360;"
    assert row in txt
    path = tmp_path / "case9_tight.m"
    path.write_text(txt.replace(row, "\t5\t6\t0.039\t0.17\t0.358\t20\t20\t20\t0\t0\t1\t-360\t360;"))
    d = dict(rho_pq=100.0, rho_va=1e4, max_outer=1, max_inner=max_inner)
    st, rep = gridadmm.solve(gridadmm.Network(str(path)), gridadmm.Config(**d))
    ref = RefCapi(oracle_mod, str(path), **d)
    rst, rrep = ref.solve()
    assert st == rst == 4
    m, rm = rep.metrics(), ref.metrics(ref.h, rrep)
    assert rm["limit_violation"] > 0.0
    for k in rm:
        assert bits(m[k]) == bits(rm[k]), (k, m[k], rm[k])
    vm, va = rep.voltages()
    rvm, rva = np.zeros_like(vm), np.zeros_like(va)
    dp = ctypes.POINTER(ctypes.c_double)
    ref.h.gridadmm_report_voltages(rrep, rvm.ctypes.data_as(dp), rva.ctypes.data_as(dp))
    assert np.array_equal(bits(vm), bits(rvm)) and np.array_equal(bits(va), bits(rva))
    sol, rsol = tmp_path / "s.json", tmp_path / "rs.json"
    rep.write_solution(str(sol))
    assert ref.h.gridadmm_report_write_solution(rrep, os.fsencode(str(rsol)), -1.0) == 0
    assert mask_wall_clock_json(sol.read_text()) == mask_wall_clock_json(rsol.read_text())
    ref.h.gridadmm_report_free(rrep)
    ref.close()


def test_full_solve_2868_shape_matches_reference(gridadmm, oracle_mod):
    """Full cold start of the 2868rte-shaped synthetic grid (BASELINE
    configs[1]) to convergence through both libraries' gridadmm_solve: status,
    iteration counts and every metric bit (the reference on all host cores,
    ~80 s on 16)."""
    from gridcases import synth
    path = synth.ensure_case("case2868rte", "/tmp/gridadmm_cases")
    d = dict(rho_pq=1000.0, rho_va=1e4)
    st, rep = gridadmm.solve(gridadmm.Network(path), gridadmm.Config(**d))
    rst, rm = oracle_mod.capi_solve(oracle_mod.ref_capi(), path, workers=os.cpu_count() or 1, **d)
    assert st == rst == 0
    m = rep.metrics()
    for k in rm:
        assert bits(m[k]) == bits(rm[k]), (k, m[k], rm[k])
