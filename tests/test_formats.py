"""File-format contracts against the reference library (no GPU): the MATPOWER
parser's error classes (proj/src/netdata.cpp:64-103 — std::stod rejects
out-of-range tokens) and the tracking-profile reader's error paths
(proj/src/tracking.cpp:114-196), which run before any device work in both
libraries.  Status codes and messages must be identical."""
import ctypes
import os

import pytest

from conftest import case_path


def _ref_load(oracle_mod, path):
    h = oracle_mod.ref_capi()
    net = ctypes.c_void_p()
    st = h.gridadmm_network_load(os.fsencode(path), ctypes.byref(net))
    msg = h.gridadmm_last_error().decode()
    if st == 0:
        h.gridadmm_network_free(net)
    return st, msg


def _my_load(gridadmm, path):
    try:
        gridadmm.Network(path).close()
        return 0, ""
    except gridadmm.GridAdmmError as e:
        return e.status, e.message


def _mutate(tmp_path, name, old, new):
    text = open(case_path("case9")).read()
    assert old in text, old
    p = tmp_path / name
    p.write_text(text.replace(old, new, 1))
    return str(p)


@pytest.fixture
def need_ref(oracle_mod):
    if not oracle_mod.have_ref():
        pytest.skip("reference oracle not built")


MUTATIONS = [
    ("overflow_entry", "1	3	0	0	0	0	1	1	0	345	1	1.1	0.9;", "1	3	0	0	0	0	1	1e400	0	345	1	1.1	0.9;"),
    ("underflow_entry", "1	3	0	0	0	0	1	1	0	345	1	1.1	0.9;", "1	3	0	0	0	0	1	1e-320	0	345	1	1.1	0.9;"),
    ("garbage_entry", "1	3	0	0	0	0	1	1	0	345	1	1.1	0.9;", "1	3	0	0	0	0	1	1x	0	345	1	1.1	0.9;"),
    ("overflow_scalar", "mpc.baseMVA = 100;", "mpc.baseMVA = 1e999;"),
    ("garbage_scalar", "mpc.baseMVA = 100;", "mpc.baseMVA = abc;"),
    ("missing_scalar", "mpc.baseMVA = 100;", "mpc.baseXXX = 100;"),
    ("negative_base", "mpc.baseMVA = 100;", "mpc.baseMVA = -5;"),
]


@pytest.mark.parametrize("name,old,new", MUTATIONS, ids=[m[0] for m in MUTATIONS])
def test_parser_error_classes_match_reference(gridadmm, oracle_mod, need_ref, tmp_path, name, old,
                                              new):
    path = _mutate(tmp_path, name + ".m", old, new)
    ref = _ref_load(oracle_mod, path)
    mine = _my_load(gridadmm, path)
    assert ref[0] in (1, 2), ref  # every mutation is rejected by the reference
    assert mine == ref


PROFILES = {
    "bad_header": "time,multiplier\n1,1.0\n",
    "empty": "",
    "header_only": "period,multiplier\n",
    "gap": "period,multiplier\n1,1.0\n3,1.0\n",
    "field_count": "period,multiplier\n1,1.0,2\n",
    "bad_number": "period,multiplier\n1,abc\n",
    "unknown_bus": "period,bus,multiplier\n1,1,1.0\n1,777,1.0\n",
    "per_bus_gap": "period,bus,multiplier\n2,1,1.0\n",
    "zero_period": "period,multiplier\n0,1.0\n1,1.0\n",
}


@pytest.mark.parametrize("name", sorted(PROFILES))
def test_profile_errors_match_reference(gridadmm, oracle_mod, need_ref, tmp_path, name):
    prof = tmp_path / (name + ".csv")
    prof.write_text(PROFILES[name])
    h = oracle_mod.ref_capi()
    rnet = ctypes.c_void_p()
    assert h.gridadmm_network_load(os.fsencode(case_path("case9")), ctypes.byref(rnet)) == 0
    c = h.gridadmm_config_new()
    trk = ctypes.c_void_p()
    rst = h.gridadmm_track_run(rnet, c, os.fsencode(str(prof)), ctypes.byref(trk))
    rmsg = h.gridadmm_last_error().decode()
    h.gridadmm_config_free(c)
    h.gridadmm_network_free(rnet)
    assert rst != 0 and not trk.value, (rst, rmsg)

    net = gridadmm.Network(case_path("case9"))
    with pytest.raises(gridadmm.GridAdmmError) as e:
        gridadmm.track(net, gridadmm.Config(), str(prof))
    assert e.value.status == rst
    assert e.value.message.split(os.fsdecode(str(tmp_path)))[0] == rmsg.split(str(tmp_path))[0]
