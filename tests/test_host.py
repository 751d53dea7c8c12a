"""Host-side checks (no GPU): the C-ABI library loads and exports every symbol
its headers declare; MATPOWER parsing, admittances and the coupling layout
are bit-identical to the reference's; config/report API contract
(proj/tests/test_capi.cpp:47-94); the synthetic case generator."""
import os
import re

import numpy as np
import pytest

from conftest import REPO, case_path

CASES = ["case2", "case9", "case30", "case118"]


def declared_symbols():
    names = []
    for h in ("gridadmm.h", "gridadmm_ext.h"):
        text = open(os.path.join(REPO, "include", "gridadmm", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(gridadmm_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(gridadmm):
    syms = declared_symbols()
    assert len(syms) >= 23
    lib = gridadmm.lib()
    for s in syms:
        assert hasattr(lib, s), s
    # the 23 reference entry points (proj/include/gridadmm/gridadmm.h:33-101)
    ref23 = [n for n in gridadmm.SYMBOLS]
    assert len(ref23) == 23 and set(ref23) <= set(syms)


def test_c_program_links_against_library(gridadmm, tmp_path):
    """A plain C caller compiled against include/gridadmm/gridadmm.h links and
    runs against libgridadmm.so (drop-in for the reference's C callers)."""
    import subprocess
    exe = tmp_path / "capi_link"
    libdir = os.path.dirname(gridadmm.LIB_PATH)
    src = os.path.join(REPO, "tests", "c", "capi_link.c")
    r = subprocess.run(["gcc", "-std=c11", "-I", os.path.join(REPO, "include"), src, "-o", str(exe),
                        "-L", libdir, "-lgridadmm", f"-Wl,-rpath,{libdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), case_path("case9")], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout, out.stderr)


def test_sqrt_le_bound_is_exact(tmp_path):
    """The compare-only trust-region test of the Cauchy search
    (ga_math.h sqrt_le_bound): y <= t(d) iff sqrt(y) <= d, t(d) maximal, on
    4M random radii across the exponent range and every y within 6 ulps of
    d*d; out-of-range and special radii fall back to the square root."""
    import subprocess
    exe = tmp_path / "sqrt_bound_check"
    src = os.path.join(REPO, "tests", "c", "sqrt_bound_check.cpp")
    inc = os.path.join(REPO, "paper_2110_06879_b200", "csrc")
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", inc, src, "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), "4000000"], capture_output=True, text=True)
    fails, checked = map(int, out.stdout.split())
    assert fails == 0 and checked > 3_000_000


def test_cauchy_radius_skip_is_sound(tmp_path):
    """The Cauchy search skips the radius test of backtracking trials at
    alpha0 * 2^-k, k >= 2, when x is inside its box (tron.cuh cauchy_point):
    on 2M random / adversarial instances that test always passes, while at
    k = 0 it fails often (the checker reaches the boundary)."""
    import subprocess
    exe = tmp_path / "cauchy_radius_check"
    src = os.path.join(REPO, "tests", "c", "cauchy_radius_check.cpp")
    inc = os.path.join(REPO, "paper_2110_06879_b200", "csrc")
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", inc, src, "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), "2000000"], capture_output=True, text=True)
    viol, k0_fail, n = map(int, out.stdout.split())
    assert viol == 0 and n == 2_000_000 and k0_fail > 10_000


def test_network_dimensions_and_errors(gridadmm):
    net = gridadmm.Network(case_path("case9"))
    assert (net.num_buses, net.num_generators, net.num_branches) == (9, 3, 9)
    assert net.num_rows == 78  # tests/test_decomp.cpp:33-39
    assert gridadmm.Network(case_path("case2")).num_rows == 10
    with pytest.raises(gridadmm.GridAdmmError) as e:
        gridadmm.Network("/no/such/case.m")
    assert e.value.status == 2 and "/no/such/case.m" in e.value.message


def test_config_contract(gridadmm):
    cfg = gridadmm.Config()
    cfg["rho_pq"] = 55.0
    assert cfg["rho_pq"] == 55.0
    cfg["max_inner"] = 123
    assert cfg["max_inner"] == 123
    for key, val in (("max_inner", 1.5), ("eps", -1.0), ("no_such_key", 1.0), ("rho_pq", np.nan)):
        with pytest.raises(gridadmm.GridAdmmError) as e:
            cfg[key] = val
        assert e.value.status == 3
    cfg.preset("case118")
    assert cfg["rho_pq"] == 100.0
    cfg.preset("case9241pegase")
    assert cfg["rho_va"] == 5e3
    with pytest.raises(gridadmm.GridAdmmError):
        cfg.preset("case_unknown")
    cfg["lambda_bound"] = 7.0
    assert cfg["lambda_bound"] == 7.0
    # defaults of SolverConfig (proj/src/driver.hpp:15-40)
    d = gridadmm.Config()
    assert (d["rho_pq"], d["rho_va"], d["beta0"], d["eps"], d["max_outer"], d["max_inner"]) == \
        (10.0, 1000.0, 1e3, 1e-4, 20, 1000)
    # branch-phase scheduling extensions (results never depend on them)
    assert (d["lane_budget"], d["lane_cap"], d["tile_budget"]) == (4, 16, 0)  # 0: no solo phase
    d["tile_budget"] = 48  # hand branches past 48 tile steps to whole-warp solves
    assert d["tile_budget"] == 48
    for key, val in (("lane_budget", 0), ("lane_cap", 0.5), ("tile_budget", -1)):
        with pytest.raises(gridadmm.GridAdmmError):
            d[key] = val


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("name", CASES)
def test_parser_matches_reference(gridadmm, oracle_mod, name):
    if not oracle_mod.have_ref():
        pytest.skip("reference oracle not built")
    mine = gridadmm.Network(case_path(name)).export()
    ref = oracle_mod.RefNet(case_path(name)).export()
    for k in ("bus", "gen", "branch"):
        assert np.array_equal(bits(mine[k]), bits(ref[k])), k
    for k in ("bus_id", "ends"):
        assert np.array_equal(mine[k], ref[k]), k
    assert mine["ref_bus"] == ref["ref_bus"]


@pytest.mark.parametrize("name", CASES)
def test_layout_matches_reference(gridadmm, oracle_mod, name):
    if not oracle_mod.have_ref():
        pytest.skip("reference oracle not built")
    c1, r1 = gridadmm.Network(case_path(name)).layout()
    c2, r2 = oracle_mod.RefNet(case_path(name)).layout()
    assert np.array_equal(c1, c2)
    assert np.array_equal(r1, r2)
    # every row is owned by exactly one bus (tests/test_decomp.cpp:59-71)
    assert np.array_equal(np.sort(r1), np.arange(len(r1)))


def test_synthetic_case_shapes_and_determinism(gridadmm, tmp_path, oracle_mod):
    from gridcases import synth
    p1 = synth.write_case("case2868rte", str(tmp_path / "a.m"), seed=5)
    p2 = synth.write_case("case2868rte", str(tmp_path / "b.m"), seed=5)
    assert open(p1).read() == open(p2).read()
    net = gridadmm.Network(p1)
    assert (net.num_buses, net.num_generators, net.num_branches) == synth.SHAPES["case2868rte"]
    if oracle_mod.have_ref():
        ref = oracle_mod.RefNet(p1).export()
        mine = net.export()
        for k in ("bus", "gen", "branch"):
            assert np.array_equal(bits(mine[k]), bits(ref[k])), k
        c1, r1 = net.layout()
        c2, r2 = oracle_mod.RefNet(p1).layout()
        assert np.array_equal(r1, r2)
