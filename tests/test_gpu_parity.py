"""GPU parity: the sm_100a path through the C ABI vs the reference oracle.

Bar: bit-exact.  Every comparison below is on the
raw IEEE-754 bits (``view(np.uint64)``), which is strictly stronger than the
north-star's 1e-8 relative per-iteration residual tolerance.
"""
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


def assert_bits_equal(a, b, what):
    ba, bb = bits(a), bits(b)
    if not np.array_equal(ba, bb):
        bad = np.nonzero(ba != bb)[0]
        k = bad[0]
        raise AssertionError(f"{what}: {bad.size} of {ba.size} differ; first at {k}: "
                             f"{np.asarray(a).ravel()[k]!r} vs {np.asarray(b).ravel()[k]!r}")


def assert_state_equal(gpu, ref, where):
    for f in FIELDS:
        assert_bits_equal(gpu[f], ref[f], f"{where}: {f}")


def make_cfg(ga, name, **over):
    d = dict(DESK[name])
    d.update(over)
    cfg = ga.Config()
    for k, v in d.items():
        cfg[k] = v
    return cfg, d


def test_device_sincos_matches_host_shim(gridadmm, oracle_mod):
    rng = np.random.default_rng(7)
    x = np.concatenate([
        rng.uniform(-4 * np.pi, 4 * np.pi, 2_000_000),
        rng.uniform(-1e-3, 1e-3, 100_000),
        rng.uniform(-1e4, 1e4, 100_000),
        np.array([0.0, -0.0, np.pi / 4, -np.pi / 4, np.pi / 2, np.pi, 2 * np.pi, 1e-300,
                  5e-324, np.inf, -np.inf, np.nan]),
    ])
    sd, cd = gridadmm.probe_sincos(x)
    sh, ch = oracle_mod.ref_sincos(x)
    assert_bits_equal(sd, sh, "sin")
    assert_bits_equal(cd, ch, "cos")


@pytest.mark.parametrize("tile", [1, 4, 8, 32])
@pytest.mark.parametrize("n", [4, 6, 2])
def test_tron_core_matches_reference(gridadmm, oracle_mod, n, tile):
    """Batched device TRON vs reference solve_one on random box QPs (convex and
    indefinite), acceptance.cpp:458-520 style, in both the one-lane (serial
    search), the 4- and 8-lane tiles and the whole-warp (speculative search) formulations."""
    rng = np.random.default_rng(100 + n)
    count = 4000
    A = rng.normal(size=(count, n, n))
    H = A @ A.transpose(0, 2, 1) / n
    H[: count // 2] += 0.1 * np.eye(n)
    H[count // 2:] -= 0.5 * np.eye(n)  # indefinite half: negative curvature paths
    g = rng.normal(size=(count, n))
    lo = -rng.uniform(0.1, 2.0, size=(count, n))
    hi = rng.uniform(0.1, 2.0, size=(count, n))
    x0 = rng.uniform(-0.5, 0.5, size=(count, n))
    Hf = np.ascontiguousarray(H.reshape(count, n * n))
    xd, sd, itd = gridadmm.probe_tron_qp(Hf, g, lo, hi, x0, tile=tile)
    xr, sr, itr = oracle_mod.ref_tron_qp(Hf, g, lo, hi, x0)
    assert np.array_equal(sd, sr)
    assert np.array_equal(itd, itr)
    assert_bits_equal(xd, xr, "tron x")


@pytest.mark.parametrize("name", ["case9", "case30", "case118"])
def test_cold_start_state(gridadmm, oracle_mod, name):
    net = gridadmm.Network(case_path(name))
    cfg, d = make_cfg(gridadmm, name)
    sess = gridadmm.Session(net, cfg)
    ref = oracle_mod.RefNet(case_path(name))
    s_ref = ref.cold_start(**d)
    assert_state_equal(sess.get_state(), s_ref, f"{name} cold start")


@pytest.mark.parametrize("name", ["case9", "case30", "case118"])
def test_phase_replay(gridadmm, oracle_mod, name):
    """Each phase from an identical state -> identical state (memcmp), for
    the first iterations and across an outer update."""
    net = gridadmm.Network(case_path(name))
    cfg, d = make_cfg(gridadmm, name)
    sess = gridadmm.Session(net, cfg)
    ref = oracle_mod.RefNet(case_path(name))
    s = ref.cold_start(**d)
    phases = ["generators", "branches", "buses", "z", "y"]
    for it in range(12):
        for p in phases:
            sess.set_state(s)
            aux_gpu = sess.phase(p)
            aux_ref = ref.phase(gridadmm.PHASES[p], s, **d)
            if p == "branches":
                assert aux_gpu == aux_ref, "branch failure count"
            assert_state_equal(sess.get_state(), s, f"{name} it {it} phase {p}")
        if it in (5, 9):
            zi = float(np.max(np.abs(s["z"])))
            prev = -1.0 if it == 5 else 0.5 * zi
            sess.set_state(s)
            sess.phase("outer", zi, prev)
            ref.phase(gridadmm.PHASES["outer"], s, z_inf=zi, prev_z_inf=prev, **d)
            assert_state_equal(sess.get_state(), s, f"{name} it {it} outer")


@pytest.mark.parametrize("name,iters", [("case9", 100), ("case30", 100), ("case118", 100)])
def test_residual_series_first_iterations(gridadmm, oracle_mod, name, iters):
    """North-star parity: per-iteration primal/dual residuals of the first
    100 iterations (bit-identical here), plus the final state."""
    net = gridadmm.Network(case_path(name))
    cfg, d = make_cfg(gridadmm, name)
    sess = gridadmm.Session(net, cfg)
    rec, _ = sess.iterate(iters)
    ref = oracle_mod.RefNet(case_path(name))
    d2 = dict(d, max_outer=1, max_inner=iters)
    series, info, fin = ref.solve(**d2)
    n = min(len(rec), len(series))
    assert len(rec) == len(series)
    assert_bits_equal(rec[:n, 0], series[:n, 2], f"{name} primal")
    assert_bits_equal(rec[:n, 1], series[:n, 3], f"{name} dual")
    assert_bits_equal(rec[:n, 2], series[:n, 4], f"{name} z_norm")
    # the reference closes its single outer iteration with update_outer unless
    # ||z||_inf <= eps (driver.cpp:224-238); do the same on the device
    z_last = float(rec[-1, 2])
    if not z_last <= d["eps"]:
        sess.phase("outer", z_last, -1.0)
    assert_state_equal(sess.get_state(), fin, f"{name} final")


def test_full_solve_case9_through_c_abi(gridadmm, oracle_mod, tmp_path):
    net = gridadmm.Network(case_path("case9"))
    cfg, d = make_cfg(gridadmm, "case9")
    st, rep = gridadmm.solve(net, cfg)
    assert st == 0
    ref = oracle_mod.RefNet(case_path("case9"))
    series, info, fin = ref.solve(**d)
    m = rep.metrics()
    assert m["inner_iterations"] == info[2]
    assert m["outer_iterations"] == info[1]
    assert m["branch_solve_failures"] == info[3]
    for k, idx in (("objective", 4), ("balance_inf", 5), ("limit_violation", 6),
                   ("bound_violation", 7), ("c_inf", 8)):
        assert_bits_equal(np.array([m[k]]), np.array([info[idx]]), k)
    conv = tmp_path / "conv.csv"
    rep.write_convergence(str(conv))
    rows = np.loadtxt(conv, delimiter=",", skiprows=1)
    assert rows.shape[0] == series.shape[0]
    assert_bits_equal(rows[:, 2:5], series[:, 2:5], "convergence.csv")


@pytest.mark.parametrize("name", ["case30", "case118", "case9"])
@pytest.mark.parametrize("lane_budget,tile_budget", [(1, 1), (1, 0), (2, 3)])
def test_branch_schedule_invariance(gridadmm, oracle_mod, name, lane_budget, tile_budget):
    """The branch phase's schedule (lane phase -> 8-lane tiles -> solo warps,
    with exact state hand-offs) must not change a bit: tiny budgets push
    nearly every branch through every phase; series and final state must
    still equal the reference's."""
    iters = 40
    net = gridadmm.Network(case_path(name))
    cfg, d = make_cfg(gridadmm, name)
    cfg["lane_budget"] = lane_budget
    cfg["tile_budget"] = tile_budget
    sess = gridadmm.Session(net, cfg)
    rec, _ = sess.iterate(iters)
    ref = oracle_mod.RefNet(case_path(name))
    series, info, fin = ref.solve(**dict(d, max_outer=1, max_inner=iters))
    assert len(rec) == len(series)
    assert_bits_equal(rec[:, 0:3], series[:, 2:5], f"{name} residuals")
    z_last = float(rec[-1, 2])
    if not z_last <= d["eps"]:
        sess.phase("outer", z_last, -1.0)
    assert_state_equal(sess.get_state(), fin, f"{name} final")


@pytest.mark.parametrize("shape,lane_budget", [("case13659pegase", 4), ("case13659pegase", 1),
                                               ("case2868rte", 2)])
def test_series_parity_synthetic_scale(gridadmm, oracle_mod, shape, lane_budget):
    """Residual series at scale (tens of thousands of branches: all three
    branch phases, both tile widths side by side in one tile kernel, the
    block-staged bus kernel with multi-block staging) vs the reference, for
    two device runs with different lane budgets."""
    from gridcases import synth
    import os
    iters = 30
    path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
    net = gridadmm.Network(path)
    cfg = gridadmm.Config(rho_pq=100.0, rho_va=1e4)
    cfg["lane_budget"] = lane_budget
    sess = gridadmm.Session(net, cfg)
    rec, _ = sess.iterate(iters)
    ref = oracle_mod.RefNet(path)
    series, _, _ = ref.solve(rho_pq=100.0, rho_va=1e4, max_outer=1, max_inner=iters,
                             workers=os.cpu_count() or 1)
    assert len(rec) == len(series) == iters
    assert_bits_equal(rec[:, 0:3], series[:, 2:5], f"{shape} residuals")


@pytest.mark.parametrize("shape,preset", [("case_ACTIVSg70k", "case_ACTIVSg70k"),
                                          ("case_ACTIVSg25k", "case_ACTIVSg25k"),
                                          ("case9241pegase", "case9241pegase")])
def test_series_parity_headline_scale(gridadmm, oracle_mod, shape, preset):
    """North-star bar at the BASELINE configs' own scale and penalties: the
    first 100 inner iterations of the cold start (preset rho, default
    tolerances) -- residual series and the whole final state bit for bit."""
    from gridcases import synth
    import os
    iters = 100
    path = synth.ensure_case(shape, "/tmp/gridadmm_cases")
    net = gridadmm.Network(path)
    rpq, rva = oracle_mod.ref_preset(preset)
    cfg = gridadmm.Config(preset)
    assert (cfg["rho_pq"], cfg["rho_va"]) == (rpq, rva)
    sess = gridadmm.Session(net, cfg)
    rec, _ = sess.iterate(iters)
    ref = oracle_mod.RefNet(path)
    series, _, fin = ref.solve(rho_pq=rpq, rho_va=rva, max_outer=1, max_inner=iters,
                               workers=os.cpu_count() or 1)
    assert len(rec) == len(series) == iters
    assert_bits_equal(rec[:, 0:3], series[:, 2:5], f"{shape} residuals")
    z_last = float(rec[-1, 2])
    if not z_last <= 1e-4:
        sess.phase("outer", z_last, -1.0)
    assert_state_equal(sess.get_state(), fin, f"{shape} state after {iters} iterations")
