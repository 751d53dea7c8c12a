"""oracle — TEST INFRASTRUCTURE ONLY (parity checker, never the product).

Two CPU checkers for the ADMM hot path, both pinned to the same sincos as the
device code (``paper_2110_06879_b200/csrc/ga_sincos.h``):

* ``_ref/libgridadmm_ref.so`` — the UNMODIFIED reference C++ solver
  (/root/reference/proj/src/*.cpp) compiled in place by ``oracle/Makefile``
  with ``sincos_shim.c`` and the phase-replay harness ``ref_harness.cpp``.
  Built in the dev container (where /root/reference exists) and shipped to the
  GPU box as a prebuilt .so.
* ``liboracle.so`` — ``gridadmm_oracle.c``, a plain-C restatement of the hot
  path (generator / branch TRON / bus / z-y / loop control), each function
  citing the reference line it follows; pinned bit-for-bit against the
  compiled reference and the golden vectors in ``tests/golden``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
and reference legs may import this package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgridadmm_ref.so")
# the same reference objects linked against glibc's own sincos (no pin)
STOCK_SO = os.path.join(HERE, "_ref", "libgridadmm_stock.so")
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SRC = "/root/reference/proj/src"

_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)
_P = ctypes.c_void_p

STATE_FIELDS = ("x", "xbar", "z", "y", "lambda", "rho", "bus_w", "bus_theta", "branch_point",
                "lt_ij", "lt_ji", "rho_tilde")


class StateView(ctypes.Structure):
    _fields_ = [(n, _DP) for n in ("x", "xbar", "z", "y", "lambda_", "rho", "bus_w", "bus_theta",
                                   "branch_point", "lt_ij", "lt_ji", "rho_tilde", "beta")]


def build(verbose: bool = False) -> None:
    """make -C oracle (C restatement always; reference .so when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + (out.stdout or "") + (out.stderr or ""))


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _dp(a):
    return None if a is None else a.ctypes.data_as(_DP)


def config_vector(rho_pq=10.0, rho_va=1000.0, beta0=1e3, eps=1e-4, inner_tol=0.0, max_outer=20,
                  max_inner=1000, workers=1, lambda_bound=1e12, beta_max=1e12):
    """Solver settings in the harness order (ref_harness.cpp config_from)."""
    return (ctypes.c_double * 10)(rho_pq, rho_va, beta0, eps, inner_tol, max_outer, max_inner,
                                  workers, lambda_bound, beta_max)


def state_shapes(nb, ng, nl):
    m = 2 * ng + 8 * nl
    return {"x": m, "xbar": m, "z": m, "y": m, "lambda": m, "rho": m, "bus_w": nb,
            "bus_theta": nb, "branch_point": 6 * nl, "lt_ij": nl, "lt_ji": nl, "rho_tilde": nl}


def make_view(arrays):
    v = StateView()
    for f in STATE_FIELDS:
        a = arrays.get(f)
        setattr(v, "lambda_" if f == "lambda" else f, _dp(a) if a is not None else None)
    b = arrays.get("beta")
    v.beta = _dp(b) if b is not None else None
    return v


class RefLib:
    """ctypes binding of _ref/libgridadmm_ref.so."""

    _h = None

    @classmethod
    def get(cls):
        if cls._h is None:
            if not have_ref():
                raise FileNotFoundError(f"{REF_SO} missing; run `make -C oracle` where "
                                        "/root/reference exists")
            h = ctypes.CDLL(REF_SO)
            h.ref_net_load.restype = _P
            h.ref_net_load.argtypes = [ctypes.c_char_p]
            h.ref_net_free.argtypes = [_P]
            h.ref_net_dims.argtypes = [_P, _IP, _IP, _IP, _IP]
            h.ref_net_export.argtypes = [_P, _DP, _IP, _DP, _IP, _DP, _IP]
            h.ref_layout_export.argtypes = [_P, _IP, _IP]
            h.ref_cold_start.argtypes = [_P, _DP, ctypes.POINTER(StateView)]
            h.ref_phase.restype = ctypes.c_long
            h.ref_phase.argtypes = [_P, ctypes.c_int, _DP, ctypes.POINTER(StateView), _D, _D]
            h.ref_solve.argtypes = [_P, _DP, ctypes.POINTER(StateView), ctypes.POINTER(StateView),
                                    _DP, ctypes.c_int, _IP, _DP]
            h.ref_tron_qp.argtypes = [ctypes.c_int, ctypes.c_int, _DP, _DP, _DP, _DP, _DP, _IP, _IP]
            h.ref_last_error.restype = ctypes.c_char_p
            h.ga_oracle_sincos.argtypes = [_D, _DP, _DP]
            h.ga_oracle_sincos_batch.argtypes = [ctypes.c_long, _DP, _DP, _DP]
            cls._h = h
        return cls._h


class RefNet:
    """A network loaded by the reference's own parser (netdata.cpp:124-237)."""

    def __init__(self, path: str):
        self.lib = RefLib.get()
        self.h = self.lib.ref_net_load(os.fsencode(path))
        if not self.h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        nb, ng, nl, m = (ctypes.c_int() for _ in range(4))
        self.lib.ref_net_dims(self.h, ctypes.byref(nb), ctypes.byref(ng), ctypes.byref(nl),
                              ctypes.byref(m))
        self.nb, self.ng, self.nl, self.m = nb.value, ng.value, nl.value, m.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_net_free(self.h)
            self.h = None

    def shapes(self):
        return state_shapes(self.nb, self.ng, self.nl)

    def empty_state(self) -> Dict[str, np.ndarray]:
        s = {k: np.zeros(n) for k, n in self.shapes().items()}
        s["beta"] = np.zeros(1)
        return s

    def export(self):
        bus = np.zeros(6 * self.nb)
        ids = np.zeros(self.nb, dtype=np.int32)
        gen = np.zeros(8 * self.ng)
        ends = np.zeros(2 * self.nl, dtype=np.int32)
        br = np.zeros(14 * self.nl)
        ref = ctypes.c_int()
        self.lib.ref_net_export(self.h, _dp(bus), ids.ctypes.data_as(_IP), _dp(gen),
                                ends.ctypes.data_as(_IP), _dp(br), ctypes.byref(ref))
        return {"bus": bus.reshape(-1, 6), "bus_id": ids, "gen": gen.reshape(-1, 8),
                "ends": ends.reshape(-1, 2), "branch": br.reshape(-1, 14), "ref_bus": ref.value}

    def layout(self):
        counts = np.zeros(6 * self.nb, dtype=np.int32)
        rows = np.zeros(max(self.m, 1), dtype=np.int32)
        self.lib.ref_layout_export(self.h, counts.ctypes.data_as(_IP), rows.ctypes.data_as(_IP))
        return counts.reshape(-1, 6), rows[: self.m]

    def cold_start(self, **cfg) -> Dict[str, np.ndarray]:
        s = self.empty_state()
        v = make_view(s)
        self.lib.ref_cold_start(self.h, config_vector(**cfg), ctypes.byref(v))
        return s

    def phase(self, phase: int, state: Dict[str, np.ndarray], z_inf=0.0, prev_z_inf=-1.0,
              **cfg) -> int:
        """Runs one reference phase on `state` in place (kernels.hpp:70-101)."""
        v = make_view(state)
        return int(self.lib.ref_phase(self.h, phase, config_vector(**cfg), ctypes.byref(v),
                                      z_inf, prev_z_inf))

    def solve(self, init: Optional[Dict[str, np.ndarray]] = None, cap: int = 100000, **cfg):
        """Full reference solve; returns (series[n, 6], info[9], final_state).
        series columns: outer, inner, primal, dual, z_norm, elapsed_s."""
        series = np.zeros(6 * cap)
        n = ctypes.c_int()
        info = np.zeros(9)
        fin = self.empty_state()
        vf = make_view(fin)
        vi = make_view(init) if init is not None else None
        rc = self.lib.ref_solve(self.h, config_vector(**cfg),
                                ctypes.byref(vi) if vi is not None else None, ctypes.byref(vf),
                                _dp(series), cap, ctypes.byref(n), _dp(info))
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        k = min(n.value, cap)
        return series[: 6 * k].reshape(-1, 6), info, fin


# The reference's C ABI (proj/include/gridadmm/gridadmm.h:33-101), typed here
# so the oracle never imports the product package.
_S, _I = ctypes.c_char_p, ctypes.c_int
REF_SYMBOLS = {
    "gridadmm_last_error": (_S, []),
    "gridadmm_network_load": (_I, [_S, ctypes.POINTER(_P)]),
    "gridadmm_network_free": (None, [_P]),
    "gridadmm_network_num_buses": (_I, [_P]),
    "gridadmm_network_num_generators": (_I, [_P]),
    "gridadmm_network_num_branches": (_I, [_P]),
    "gridadmm_config_new": (_P, []),
    "gridadmm_config_free": (None, [_P]),
    "gridadmm_config_set": (_I, [_P, _S, _D]),
    "gridadmm_config_get": (_I, [_P, _S, _DP]),
    "gridadmm_config_preset": (_I, [_P, _S]),
    "gridadmm_solve": (_I, [_P, _P, ctypes.POINTER(_P)]),
    "gridadmm_report_free": (None, [_P]),
    "gridadmm_report_metric": (_I, [_P, _S, _DP]),
    "gridadmm_report_dispatch": (_I, [_P, _DP, _DP]),
    "gridadmm_report_voltages": (_I, [_P, _DP, _DP]),
    "gridadmm_report_write_solution": (_I, [_P, _S, _D]),
    "gridadmm_report_write_convergence": (_I, [_P, _S]),
    "gridadmm_track_run": (_I, [_P, _P, _S, ctypes.POINTER(_P)]),
    "gridadmm_track_free": (None, [_P]),
    "gridadmm_track_num_periods": (_I, [_P]),
    "gridadmm_track_period_report": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "gridadmm_track_write_periods": (_I, [_P, _S, _DP, _I]),
}
METRIC_KEYS = ("objective", "balance_inf", "limit_violation", "bound_violation", "c_inf",
               "outer_iterations", "inner_iterations", "branch_solve_failures")


def ref_capi():
    """The reference's own C ABI (the 23 gridadmm_* symbols of
    proj/include/gridadmm/gridadmm.h) from _ref/libgridadmm_ref.so."""
    h = RefLib.get()
    for name, (res, args) in REF_SYMBOLS.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


_STOCK = None


def have_stock() -> bool:
    return os.path.exists(STOCK_SO)


def stock_capi():
    """The reference's C ABI from _ref/libgridadmm_stock.so: the unmodified
    reference with glibc's sincos (host-dependent bits; compared with the
    pinned build and the product at tolerance only)."""
    global _STOCK
    if _STOCK is None:
        h = ctypes.CDLL(STOCK_SO)
        for name, (res, args) in REF_SYMBOLS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _STOCK = h
    return _STOCK


def capi_solve(h, case_path: str, **cfg):
    """gridadmm_solve through a reference C ABI handle; returns (status, metrics)."""
    net = ctypes.c_void_p()
    assert h.gridadmm_network_load(os.fsencode(case_path), ctypes.byref(net)) == 0
    c = h.gridadmm_config_new()
    for k, v in cfg.items():
        assert h.gridadmm_config_set(c, k.encode(), float(v)) == 0, k
    rep = ctypes.c_void_p()
    st = h.gridadmm_solve(net, c, ctypes.byref(rep))
    m = ref_metrics(h, rep) if rep.value else {}
    if rep.value:
        h.gridadmm_report_free(rep)
    h.gridadmm_config_free(c)
    h.gridadmm_network_free(net)
    return st, m


def ref_metrics(h, rep) -> Dict[str, float]:
    out = {}
    for key in METRIC_KEYS:
        v = ctypes.c_double()
        h.gridadmm_report_metric(rep, key.encode(), ctypes.byref(v))
        out[key] = v.value
    return out


def ref_preset(name: str):
    """(rho_pq, rho_va) of a named preset, from the reference's own table
    (capi.cpp:25-39) through gridadmm_config_preset."""
    h = ref_capi()
    c = h.gridadmm_config_new()
    try:
        if h.gridadmm_config_preset(c, name.encode()) != 0:
            raise KeyError(name)
        out = []
        for key in ("rho_pq", "rho_va"):
            v = ctypes.c_double()
            h.gridadmm_config_get(c, key.encode(), ctypes.byref(v))
            out.append(v.value)
        return tuple(out)
    finally:
        h.gridadmm_config_free(c)


def ref_track(case_path: str, profile_csv: str, preset: str, **cfg):
    """gridadmm_track_run through the reference's C ABI; returns a list of
    per-period metric dicts and the status."""
    h = ref_capi()
    net = ctypes.c_void_p()
    assert h.gridadmm_network_load(os.fsencode(case_path), ctypes.byref(net)) == 0
    c = h.gridadmm_config_new()
    assert h.gridadmm_config_preset(c, preset.encode()) == 0
    for k, v in cfg.items():
        assert h.gridadmm_config_set(c, k.encode(), float(v)) == 0, k
    trk = ctypes.c_void_p()
    st = h.gridadmm_track_run(net, c, os.fsencode(profile_csv), ctypes.byref(trk))
    out = []
    if not trk.value:
        h.gridadmm_config_free(c)
        h.gridadmm_network_free(net)
        return st, out
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        csv = os.path.join(td, "periods.csv")
        assert h.gridadmm_track_write_periods(trk, os.fsencode(csv), None, 0) == 0
        times = np.genfromtxt(csv, delimiter=",", names=True, ndmin=1)["time_s"]
    for p in range(1, h.gridadmm_track_num_periods(trk) + 1):
        rep = ctypes.c_void_p()
        assert h.gridadmm_track_period_report(trk, p, ctypes.byref(rep)) == 0
        m = ref_metrics(h, rep)
        m["time_s"] = float(times[p - 1])
        out.append(m)
        h.gridadmm_report_free(rep)
    h.gridadmm_track_free(trk)
    h.gridadmm_config_free(c)
    h.gridadmm_network_free(net)
    return st, out


class OracleNet(ctypes.Structure):
    _fields_ = [("nb", ctypes.c_int), ("ng", ctypes.c_int), ("nl", ctypes.c_int),
                ("ref_bus", ctypes.c_int), ("bus", _DP), ("gen", _DP), ("ends", _IP),
                ("branch", _DP)]


class PortLib:
    """ctypes binding of liboracle.so (the C restatement)."""

    _h = None

    @classmethod
    def get(cls):
        if cls._h is None:
            if not os.path.exists(PORT_SO):
                build()
            h = ctypes.CDLL(PORT_SO)
            h.oracle_cold_start.argtypes = [ctypes.POINTER(OracleNet), _DP, ctypes.POINTER(StateView)]
            h.oracle_phase.restype = ctypes.c_long
            h.oracle_phase.argtypes = [ctypes.POINTER(OracleNet), ctypes.c_int, _DP,
                                       ctypes.POINTER(StateView), _D, _D]
            h.oracle_solve.argtypes = [ctypes.POINTER(OracleNet), _DP, ctypes.POINTER(StateView),
                                       ctypes.POINTER(StateView), _DP, ctypes.c_int, _IP, _DP]
            h.oracle_census.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
            cls._h = h
        return cls._h


def export_network(path: str):
    """Flat network arrays for the C restatement: parsed by the reference's
    own parser when oracle/_ref is present, else by the product parser (which
    tests/test_host.py pins to the reference bit-for-bit)."""
    if have_ref():
        return RefNet(path).export()
    import paper_2110_06879_b200 as ga
    return ga.Network(path).export()


class PortNet:
    """The C restatement (gridadmm_oracle.c) on one network."""

    def __init__(self, path: str):
        self.lib = PortLib.get()
        ex = export_network(path)
        self.arrays = {
            "bus": np.ascontiguousarray(ex["bus"].ravel()),
            "gen": np.ascontiguousarray(ex["gen"].ravel()),
            "ends": np.ascontiguousarray(ex["ends"].ravel().astype(np.int32)),
            "branch": np.ascontiguousarray(ex["branch"].ravel()),
        }
        self.nb, self.ng, self.nl = len(ex["bus"]), len(ex["gen"]), len(ex["ends"])
        self.m = 2 * self.ng + 8 * self.nl
        a = self.arrays
        self.net = OracleNet(self.nb, self.ng, self.nl, ex["ref_bus"], _dp(a["bus"]), _dp(a["gen"]),
                             a["ends"].ctypes.data_as(_IP), _dp(a["branch"]))

    def empty_state(self):
        s = {k: np.zeros(n) for k, n in state_shapes(self.nb, self.ng, self.nl).items()}
        s["beta"] = np.zeros(1)
        return s

    def cold_start(self, **cfg):
        s = self.empty_state()
        v = make_view(s)
        self.lib.oracle_cold_start(ctypes.byref(self.net), config_vector(**cfg), ctypes.byref(v))
        return s

    def phase(self, phase, state, z_inf=0.0, prev_z_inf=-1.0, **cfg):
        v = make_view(state)
        return int(self.lib.oracle_phase(ctypes.byref(self.net), phase, config_vector(**cfg),
                                         ctypes.byref(v), z_inf, prev_z_inf))

    def solve(self, init=None, cap=100000, **cfg):
        series = np.zeros(6 * cap)
        n = ctypes.c_int()
        info = np.zeros(9)
        fin = self.empty_state()
        vf = make_view(fin)
        vi = make_view(init) if init is not None else None
        rc = self.lib.oracle_solve(ctypes.byref(self.net), config_vector(**cfg),
                                   ctypes.byref(vi) if vi is not None else None, ctypes.byref(vf),
                                   _dp(series), cap, ctypes.byref(n), _dp(info))
        if rc != 0:
            raise RuntimeError("oracle solve failed (singular bus)")
        k = min(n.value, cap)
        return series[: 6 * k].reshape(-1, 6), info, fin

    def census(self, reset=True):
        out = (ctypes.c_ulonglong * 6)()
        self.lib.oracle_census(out, 1 if reset else 0)
        return list(out)


def ref_tron_qp(H, g, lo, hi, x0):
    lib = RefLib.get()
    count, n = g.shape
    x = np.ascontiguousarray(x0, dtype=np.float64).copy()
    st = np.zeros(count, dtype=np.int32)
    its = np.zeros(count, dtype=np.int32)
    args = [np.ascontiguousarray(a, dtype=np.float64) for a in (H, g, lo, hi)]
    lib.ref_tron_qp(count, n, *[_dp(a) for a in args], _dp(x), st.ctypes.data_as(_IP),
                    its.ctypes.data_as(_IP))
    return x, st, its


def ref_sincos(x):
    lib = RefLib.get()
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.zeros_like(x)
    c = np.zeros_like(x)
    lib.ga_oracle_sincos_batch(x.size, _dp(x), _dp(s), _dp(c))
    return s, c
