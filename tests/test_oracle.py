"""The C restatement oracle (oracle/gridadmm_oracle.c) pinned against the
compiled reference (oracle/_ref, when present) and the committed golden
vectors (tests/golden, generated from the reference by
scripts/make_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, case_path

DESK = {  # proj/tests/acceptance.cpp:58-69
    "case9": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5),
    "case30": dict(rho_pq=100.0, rho_va=1e4, eps=1e-5),
    "case118": dict(rho_pq=100.0, rho_va=1e4, eps=1e-6, max_inner=300),
}
FIELDS = ("x", "xbar", "z", "y", "lambda", "rho", "bus_w", "bus_theta", "branch_point", "lt_ij",
          "lt_ji", "rho_tilde", "beta")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("name", ["case9", "case30", "case118"])
def test_port_matches_golden_series(oracle_mod, name):
    gold = np.load(os.path.join(GOLDEN, f"series_{name}.npz"))
    port = oracle_mod.PortNet(case_path(name))
    n = int(gold["iters"])
    series, info, fin = port.solve(**dict(DESK[name], max_outer=1, max_inner=n))
    assert series.shape[0] == gold["series"].shape[0]
    assert same(series[:, 2:5], gold["series"][:, 2:5])
    for f in ("x", "xbar", "z", "y", "branch_point", "lt_ij", "lt_ji", "rho_tilde", "lambda"):
        assert same(fin[f], gold[f]), f


@pytest.mark.parametrize("name", ["case9", "case30", "case118"])
def test_port_phases_match_reference(oracle_mod, name):
    if not oracle_mod.have_ref():
        pytest.skip("reference oracle not built")
    ref = oracle_mod.RefNet(case_path(name))
    port = oracle_mod.PortNet(case_path(name))
    d = DESK[name]
    s_ref = ref.cold_start(**d)
    s_port = port.cold_start(**d)
    for f in FIELDS:
        assert same(s_ref[f], s_port[f]), f"cold start {f}"
    for it in range(6):
        for p in range(5):
            r1 = ref.phase(p, s_ref, **d)
            r2 = port.phase(p, s_port, **d)
            if p in (1, 2):
                assert r1 == r2
            for f in FIELDS:
                assert same(s_ref[f], s_port[f]), f"it {it} phase {p} {f}"


def test_port_full_solve_case9_matches_golden(oracle_mod):
    gold = json.load(open(os.path.join(GOLDEN, "solve_case9.json")))
    port = oracle_mod.PortNet(case_path("case9"))
    series, info, fin = port.solve(**DESK["case9"])
    assert int(info[0]) == gold["status"]
    assert int(info[1]) == gold["outer_iterations"]
    assert int(info[2]) == gold["inner_iterations"]
    last = series[-1, 2:5]
    assert same(last, np.array(gold["last_record"]))


def test_port_census_counts_work(oracle_mod):
    port = oracle_mod.PortNet(case_path("case30"))
    port.census(reset=True)
    port.solve(**dict(DESK["case30"], max_outer=1, max_inner=5))
    c = port.census(reset=True)
    assert c[0] > 0 and c[2] > 0  # flops and 6-var TRON iterations (case30 is rate-limited)
    assert 1000 < c[4] / c[2] < 10000  # flops per 6-var TRON iteration
