"""Warm-start tracking parity (north-star (d), tracking.cpp:30-85): the
device-resident carry-over between load snapshots vs the reference's
gridadmm_track_run on the same profile — identical per-period iteration
counts and bit-identical objectives / violations."""
import numpy as np
import pytest

from conftest import case_path

pytestmark = pytest.mark.gpu


def bits(v):
    return np.float64(v).view(np.uint64)


@pytest.mark.parametrize("name,profile,extra", [
    ("case9", "period,multiplier\n1,1.0\n2,1.005\n3,1.0\n", dict(eps=1e-4)),
    ("case30", "period,multiplier\n1,1.0\n2,1.005\n3,1.010\n4,1.015\n", dict(eps=1e-5)),
])
def test_tracking_matches_reference(gridadmm, oracle_mod, tmp_path, name, profile, extra):
    csv = tmp_path / "profile.csv"
    csv.write_text(profile)
    net = gridadmm.Network(case_path(name))
    cfg = gridadmm.Config(name, **extra)
    st, trk = gridadmm.track(net, cfg, str(csv))
    ref_st, ref = oracle_mod.ref_track(case_path(name), str(csv), name, **extra)
    assert st == ref_st
    assert trk.num_periods == len(ref)
    for p, rm in enumerate(ref, start=1):
        m = trk.period_report(p).metrics()
        for key in ("inner_iterations", "outer_iterations", "branch_solve_failures"):
            assert m[key] == rm[key], (p, key)
        for key in ("objective", "c_inf", "balance_inf", "limit_violation", "bound_violation"):
            assert bits(m[key]) == bits(rm[key]), (p, key, m[key], rm[key])


def test_tracking_per_bus_profile_and_ramp(gridadmm, oracle_mod, tmp_path):
    """Per-bus multipliers (period,bus,multiplier) and the ramp windows of
    later periods (tracking.cpp:48-70)."""
    net = gridadmm.Network(case_path("case9"))
    ids = net.export()["bus_id"]
    lines = ["period,bus,multiplier"]
    rng = np.random.default_rng(3)
    for t in (1, 2, 3):
        for i in ids:
            lines.append(f"{t},{i},{1.0 + 0.01 * (t - 1) + 0.002 * rng.standard_normal():.6f}")
    csv = tmp_path / "perbus.csv"
    csv.write_text("\n".join(lines) + "\n")
    cfg = gridadmm.Config("case9", eps=1e-4, ramp_frac=0.05)
    st, trk = gridadmm.track(net, cfg, str(csv))
    ref_st, ref = oracle_mod.ref_track(case_path("case9"), str(csv), "case9", eps=1e-4, ramp_frac=0.05)
    assert st == ref_st
    for p, rm in enumerate(ref, start=1):
        m = trk.period_report(p).metrics()
        assert m["inner_iterations"] == rm["inner_iterations"]
        assert bits(m["objective"]) == bits(rm["objective"])


def test_empty_ramp_window_is_infeasible_ramp(gridadmm, oracle_mod, tmp_path):
    """RampError -> GRIDADMM_ERR_INFEASIBLE_RAMP (tracking.cpp:48-60,
    capi.cpp:302-303): a generator with pmax < 0 has ramp window
    [prev + |r|, prev - |r|] in period 2, empty for any prev_pg.  Same status,
    same message, no tracking handle."""
    import ctypes
    src = open(case_path("case9")).read()
    row = "\t3\t85\t-10.95\t300\t-300\t1.025\t100\t1\t270\t10\t"
    assert row in src
    case = tmp_path / "case9_negpmax.m"
    case.write_text(src.replace(row, "\t3\t-15\t-10.95\t300\t-300\t1.025\t100\t1\t-10\t-20\t"))
    csv = tmp_path / "profile.csv"
    csv.write_text("period,multiplier\n1,1.0\n2,1.01\n")
    extra = dict(eps=1e-4, max_outer=2, max_inner=40)
    net = gridadmm.Network(str(case))
    cfg = gridadmm.Config("case9", **extra)
    h = ctypes.c_void_p()
    st = gridadmm.lib().gridadmm_track_run(net.handle, cfg.handle, str(csv).encode(), ctypes.byref(h))
    msg = gridadmm.lib().gridadmm_last_error().decode()
    ref_st, ref = oracle_mod.ref_track(str(case), str(csv), "case9", **extra)
    ref_msg = oracle_mod.ref_capi().gridadmm_last_error().decode()
    assert st == ref_st == 6, (st, ref_st, msg, ref_msg)  # GRIDADMM_ERR_INFEASIBLE_RAMP
    assert not h.value and ref == []
    assert msg == ref_msg, (msg, ref_msg)
    assert "empty ramp window for generator 2 in period 2" in msg
