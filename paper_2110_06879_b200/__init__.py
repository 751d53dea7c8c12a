"""paper_2110_06879_b200 — B200-native gridadmm (component-based two-level ADMM
for AC optimal power flow, arXiv 2110.06879).

The product is ``libgridadmm.so`` (C ABI in ``include/gridadmm/gridadmm.h`` +
``gridadmm_ext.h``): a C++ host driver over hand-written sm_100a kernels.  This
module is a thin ctypes binding over that library so tests and the benchmark
call exactly what a C caller of the reference (proj/include/gridadmm/
gridadmm.h) would call.  There is no CPU fallback: importing works without the
library, but every call raises ``LibraryMissing`` until ``build()`` has produced
it, and every compute call fails loudly without a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional, Sequence

import numpy as np

__all__ = [
    "LIB_PATH", "build", "lib", "GridAdmmError", "LibraryMissing", "Network", "Config",
    "Report", "Tracking", "Session", "solve", "track", "STATUS", "PHASES",
]

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("GRIDADMM_LIB", os.path.join(PKG_DIR, "libgridadmm.so"))

STATUS = {
    0: "OK", 1: "ERR_IO", 2: "ERR_PARSE", 3: "ERR_INVALID_ARG", 4: "ERR_ITERATION_LIMIT",
    5: "ERR_DIVERGED", 6: "ERR_INFEASIBLE_RAMP", 7: "ERR_INTERNAL",
}
PHASES = {"generators": 0, "branches": 1, "buses": 2, "z": 3, "y": 4, "outer": 5}

# gridadmm.h symbol table: name -> (restype, argtypes)
_P = ctypes.c_void_p
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)
_S = ctypes.c_char_p
_I = ctypes.c_int


class StateView(ctypes.Structure):
    """gridadmm_state_view (gridadmm_ext.h)."""
    _fields_ = [(n, _DP) for n in ("x", "xbar", "z", "y", "lambda_", "rho", "bus_w", "bus_theta",
                                   "branch_point", "lt_ij", "lt_ji", "rho_tilde", "beta")]


SYMBOLS = {
    # the 23 reference entry points (proj/include/gridadmm/gridadmm.h:33-101)
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
EXT_SYMBOLS = {
    "gridadmm_network_num_rows": (_I, [_P]),
    "gridadmm_network_export": (_I, [_P, _DP, _IP, _DP, _IP, _DP, _IP]),
    "gridadmm_network_layout": (_I, [_P, _IP, _IP]),
    "gridadmm_network_partition": (_I, [_P, _I, _IP]),
    "gridadmm_network_set_branch_weights": (_I, [_P, _IP]),
    "gridadmm_network_exchange_rows": (_I, [_P, _I, _I, _I, _IP, _IP, _IP, _IP]),
    "gridadmm_session_new": (_I, [_P, _P, ctypes.POINTER(_P)]),
    "gridadmm_session_free": (None, [_P]),
    "gridadmm_session_solve": (_I, [_P, _P, _I, ctypes.POINTER(_P)]),
    "gridadmm_nccl_unique_id": (_I, [ctypes.c_char_p]),
    "gridadmm_session_new_dist": (_I, [_P, _P, _I, _I, ctypes.c_char_p, ctypes.POINTER(_P)]),
    "gridadmm_session_get_state": (_I, [_P, ctypes.POINTER(StateView)]),
    "gridadmm_session_set_state": (_I, [_P, ctypes.POINTER(StateView)]),
    "gridadmm_session_phase": (_I, [_P, _I, _DP]),
    "gridadmm_session_iterate": (_I, [_P, _I, _DP, _IP, _IP]),
    "gridadmm_session_timed_steps": (_I, [_P, _I, ctypes.c_size_t, _DP, _DP]),
    "gridadmm_session_kernel_time":(_I, [_P, _I, _DP, ctypes.POINTER(ctypes.c_longlong)]),
    "gridadmm_session_counters": (_I, [_P, ctypes.POINTER(ctypes.c_longlong),
                                       ctypes.POINTER(ctypes.c_longlong)]),
    "gridadmm_device_count": (_I, []),
    "gridadmm_session_branch_costs": (_I, [_P, _IP]),
    "gridadmm_session_step_counters": (_I, [_P, ctypes.POINTER(ctypes.c_longlong)]),
    "gridadmm_debug_tron_stats": (_I, [ctypes.POINTER(ctypes.c_ulonglong), _I]),
    "gridadmm_probe_tron_qp": (_I, [_I, _I, _DP, _DP, _DP, _DP, _DP, _IP, _IP, _I]),
    "gridadmm_probe_sincos": (_I, [_I, _DP, _DP, _DP]),
    "gridadmm_probe_fp64_peak": (_I, [_I, _DP, _DP]),
}


class LibraryMissing(RuntimeError):
    pass


class GridAdmmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


def build(verbose: bool = False) -> str:
    """Compile libgridadmm.so in-tree (sm_100a); returns its path."""
    out = subprocess.run(["make", "-C", os.path.join(PKG_DIR, "csrc"), "-j8"],
                         capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("libgridadmm build failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


_LIB: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(f"{LIB_PATH} not built; run paper_2110_06879_b200.build()")
        h = ctypes.CDLL(LIB_PATH)
        for table in (SYMBOLS, EXT_SYMBOLS):
            for name, (res, args) in table.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
        _LIB = h
    return _LIB


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_DP)


def _check(status: int, allow=(0,)) -> int:
    if status not in allow:
        raise GridAdmmError(status, lib().gridadmm_last_error().decode())
    return status


class Network:
    """gridadmm_network: a parsed MATPOWER case (reference netdata.cpp:124-237)."""

    def __init__(self, path: str):
        h = _P()
        _check(lib().gridadmm_network_load(os.fsencode(path), ctypes.byref(h)))
        self._h = h
        self.path = path

    @property
    def handle(self):
        return self._h

    @property
    def num_buses(self) -> int:
        return lib().gridadmm_network_num_buses(self._h)

    @property
    def num_generators(self) -> int:
        return lib().gridadmm_network_num_generators(self._h)

    @property
    def num_branches(self) -> int:
        return lib().gridadmm_network_num_branches(self._h)

    @property
    def num_rows(self) -> int:
        return lib().gridadmm_network_num_rows(self._h)

    def export(self):
        nb, ng, nl = self.num_buses, self.num_generators, self.num_branches
        bus = np.zeros(6 * nb)
        ids = np.zeros(nb, dtype=np.int32)
        gen = np.zeros(8 * ng)
        ends = np.zeros(2 * nl, dtype=np.int32)
        br = np.zeros(14 * nl)
        ref = ctypes.c_int()
        _check(lib().gridadmm_network_export(self._h, _dp(bus), ids.ctypes.data_as(_IP), _dp(gen),
                                             ends.ctypes.data_as(_IP), _dp(br), ctypes.byref(ref)))
        return {"bus": bus.reshape(-1, 6), "bus_id": ids, "gen": gen.reshape(-1, 8),
                "ends": ends.reshape(-1, 2), "branch": br.reshape(-1, 14), "ref_bus": ref.value}

    def partition(self, k: int) -> np.ndarray:
        """part_of_bus of the deterministic k-way partition (gridadmm_network_partition)."""
        out = np.zeros(max(1, self.num_buses), dtype=np.int32)
        _check(lib().gridadmm_network_partition(self._h, k, out.ctypes.data_as(_IP)))
        return out[: self.num_buses]

    def set_branch_weights(self, weights) -> None:
        """Per-branch partition weights, e.g. Session.branch_costs() of a
        previous sweep (gridadmm_network_set_branch_weights); None restores
        the class weights."""
        if weights is None:
            _check(lib().gridadmm_network_set_branch_weights(self._h, None))
            return
        w = np.ascontiguousarray(weights, dtype=np.int32)
        if w.shape != (self.num_branches,):
            raise ValueError("one weight per branch")
        _check(lib().gridadmm_network_set_branch_weights(self._h, w.ctypes.data_as(_IP)))

    def exchange_rows(self, k: int, p: int, q: int):
        """(send, recv) row lists of part p toward peer q (gridadmm_network_exchange_rows)."""
        ns, nr = ctypes.c_int(), ctypes.c_int()
        _check(lib().gridadmm_network_exchange_rows(self._h, k, p, q, None, ctypes.byref(ns), None,
                                                    ctypes.byref(nr)))
        send = np.zeros(max(ns.value, 1), dtype=np.int32)
        recv = np.zeros(max(nr.value, 1), dtype=np.int32)
        _check(lib().gridadmm_network_exchange_rows(self._h, k, p, q, send.ctypes.data_as(_IP),
                                                    ctypes.byref(ns), recv.ctypes.data_as(_IP),
                                                    ctypes.byref(nr)))
        return send[:ns.value], recv[:nr.value]

    def layout(self):
        counts = np.zeros(6 * self.num_buses, dtype=np.int32)
        rows = np.zeros(max(self.num_rows, 1), dtype=np.int32)
        _check(lib().gridadmm_network_layout(self._h, counts.ctypes.data_as(_IP),
                                             rows.ctypes.data_as(_IP)))
        return counts.reshape(-1, 6), rows[: self.num_rows]

    def close(self):
        if getattr(self, "_h", None):
            lib().gridadmm_network_free(self._h)
            self._h = None

    __del__ = close


class Config:
    """gridadmm_config (reference capi.cpp:92-173)."""

    def __init__(self, preset: Optional[str] = None, **kw):
        self._h = lib().gridadmm_config_new()
        if preset:
            _check(lib().gridadmm_config_preset(self._h, preset.encode()))
        for k, v in kw.items():
            self[k] = v

    @property
    def handle(self):
        return self._h

    def __setitem__(self, key: str, value: float):
        _check(lib().gridadmm_config_set(self._h, key.encode(), float(value)))

    def __getitem__(self, key: str) -> float:
        out = _D()
        _check(lib().gridadmm_config_get(self._h, key.encode(), ctypes.byref(out)))
        return out.value

    def preset(self, name: str):
        _check(lib().gridadmm_config_preset(self._h, name.encode()))

    def close(self):
        if getattr(self, "_h", None):
            lib().gridadmm_config_free(self._h)
            self._h = None

    __del__ = close


METRIC_KEYS = ("objective", "balance_inf", "limit_violation", "bound_violation", "c_inf",
               "outer_iterations", "inner_iterations", "branch_solve_failures")


class Report:
    """gridadmm_report (reference capi.cpp:211-273)."""

    def __init__(self, handle, net_dims):
        self._h = handle
        self._ng, self._nb = net_dims

    def metric(self, key: str) -> float:
        out = _D()
        _check(lib().gridadmm_report_metric(self._h, key.encode(), ctypes.byref(out)))
        return out.value

    def metrics(self) -> Dict[str, float]:
        return {k: self.metric(k) for k in METRIC_KEYS}

    def dispatch(self):
        pg = np.zeros(self._ng)
        qg = np.zeros(self._ng)
        _check(lib().gridadmm_report_dispatch(self._h, _dp(pg), _dp(qg)))
        return pg, qg

    def voltages(self):
        vm = np.zeros(self._nb)
        va = np.zeros(self._nb)
        _check(lib().gridadmm_report_voltages(self._h, _dp(vm), _dp(va)))
        return vm, va

    def write_solution(self, path: str, ref_objective: float = -1.0):
        _check(lib().gridadmm_report_write_solution(self._h, os.fsencode(path), ref_objective))

    def write_convergence(self, path: str):
        _check(lib().gridadmm_report_write_convergence(self._h, os.fsencode(path)))

    def close(self):
        if getattr(self, "_h", None):
            lib().gridadmm_report_free(self._h)
            self._h = None

    __del__ = close


def solve(net: Network, cfg: Config):
    """gridadmm_solve.  Returns (status, Report); status 0/4/5 carry a report."""
    h = _P()
    st = lib().gridadmm_solve(net.handle, cfg.handle, ctypes.byref(h))
    _check(st, allow=(0, 4, 5))
    return st, Report(h, (net.num_generators, net.num_buses))


class Tracking:
    def __init__(self, handle, net: Network):
        self._h = handle
        self._dims = (net.num_generators, net.num_buses)

    @property
    def num_periods(self) -> int:
        return lib().gridadmm_track_num_periods(self._h)

    def period_report(self, period: int) -> Report:
        h = _P()
        _check(lib().gridadmm_track_period_report(self._h, period, ctypes.byref(h)))
        return Report(h, self._dims)

    def write_periods(self, path: str, refs: Optional[Sequence[float]] = None):
        arr = np.asarray(refs if refs is not None else [], dtype=np.float64)
        _check(lib().gridadmm_track_write_periods(self._h, os.fsencode(path),
                                                  _dp(arr) if arr.size else None, int(arr.size)))

    def period_table(self):
        """Per-period rows of periods.csv (outputs.cpp:122-135): period,
        inner iterations, solve seconds, c_inf."""
        import tempfile
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "periods.csv")
            self.write_periods(path)
            rows = np.genfromtxt(path, delimiter=",", names=True, ndmin=1)
        return [{"period": int(r["period"]), "inner": int(r["inner_iters"]),
                 "time_s": float(r["time_s"]), "c_inf": float(r["viol_inf"])} for r in rows]

    def close(self):
        if getattr(self, "_h", None):
            lib().gridadmm_track_free(self._h)
            self._h = None

    __del__ = close


def track(net: Network, cfg: Config, profile_csv: str):
    """gridadmm_track_run.  Returns (status, Tracking or None)."""
    h = _P()
    st = lib().gridadmm_track_run(net.handle, cfg.handle, os.fsencode(profile_csv), ctypes.byref(h))
    if h.value:
        return st, Tracking(h, net)
    _check(st)
    return st, None


STATE_FIELDS = ("x", "xbar", "z", "y", "lambda", "rho", "bus_w", "bus_theta", "branch_point",
                "lt_ij", "lt_ji", "rho_tilde")


def state_shapes(nb: int, ng: int, nl: int) -> Dict[str, int]:
    m = 2 * ng + 8 * nl
    return {"x": m, "xbar": m, "z": m, "y": m, "lambda": m, "rho": m, "bus_w": nb,
            "bus_theta": nb, "branch_point": 6 * nl, "lt_ij": nl, "lt_ji": nl, "rho_tilde": nl}


def make_view(arrays: Dict[str, np.ndarray]) -> StateView:
    v = StateView()
    for f in STATE_FIELDS:
        a = arrays.get(f)
        setattr(v, "lambda_" if f == "lambda" else f, _dp(a) if a is not None else None)
    b = arrays.get("beta")
    v.beta = _dp(b) if b is not None else None
    return v


class Session:
    """Device-resident solver state (gridadmm_ext.h): phase replay + bench."""

    def __init__(self, net: Network, cfg: Config, _handle=None):
        h = _handle if _handle is not None else _P()
        if _handle is None:
            _check(lib().gridadmm_session_new(net.handle, cfg.handle, ctypes.byref(h)))
        self._h = h
        self._dims = (net.num_generators, net.num_buses)
        self.shapes = state_shapes(net.num_buses, net.num_generators, net.num_branches)

    @classmethod
    def distributed(cls, net: Network, cfg: Config, rank: int, world: int, nccl_id: bytes):
        """Rank `rank` of a `world`-process bus-graph partition (NCCL exchange)."""
        h = _P()
        _check(lib().gridadmm_session_new_dist(net.handle, cfg.handle, rank, world, nccl_id,
                                               ctypes.byref(h)))
        return cls(net, cfg, _handle=h)

    def solve(self, cfg: Config, warm: bool = True):
        """Algorithm 1 on this session's device state (gridadmm_session_solve):
        warm=True continues from the current state.  Returns (status, Report)."""
        rep = _P()
        st = lib().gridadmm_session_solve(self._h, cfg.handle, int(warm), ctypes.byref(rep))
        if not rep:
            _check(st)
        return st, Report(rep, self._dims)

    def get_state(self) -> Dict[str, np.ndarray]:
        arrs = {k: np.zeros(n) for k, n in self.shapes.items()}
        arrs["beta"] = np.zeros(1)
        v = make_view(arrs)
        _check(lib().gridadmm_session_get_state(self._h, ctypes.byref(v)))
        return arrs

    def set_state(self, arrays: Dict[str, np.ndarray]):
        keep = {k: np.ascontiguousarray(a, dtype=np.float64) for k, a in arrays.items()}
        v = make_view(keep)
        _check(lib().gridadmm_session_set_state(self._h, ctypes.byref(v)))

    def phase(self, phase, z_inf: float = 0.0, prev_z_inf: float = -1.0) -> float:
        p = PHASES[phase] if isinstance(phase, str) else int(phase)
        aux = np.array([z_inf, prev_z_inf], dtype=np.float64)
        _check(lib().gridadmm_session_phase(self._h, p, _dp(aux)))
        return float(aux[0])

    def iterate(self, n: int):
        rec = np.zeros(5 * max(n, 1))
        done = ctypes.c_int()
        stop = ctypes.c_int()
        _check(lib().gridadmm_session_iterate(self._h, n, _dp(rec), ctypes.byref(done),
                                              ctypes.byref(stop)))
        return rec[: 5 * done.value].reshape(-1, 5), stop.value

    def timed_steps(self, n: int, flush_bytes: int = 0):
        """n iterations, per-step device ms (CUDA events on the session stream)."""
        ms = np.zeros(max(n, 1))
        rec = np.zeros(5 * max(n, 1))
        _check(lib().gridadmm_session_timed_steps(self._h, n, flush_bytes, _dp(ms), _dp(rec)))
        return ms[:n], rec[: 5 * n].reshape(-1, 5)

    def kernel_time(self, cls: int):
        ms = _D()
        n = ctypes.c_longlong()
        _check(lib().gridadmm_session_kernel_time(self._h, cls, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def branch_costs(self) -> np.ndarray:
        out = np.zeros(max(1, self.shapes["lt_ij"]), dtype=np.int32)
        _check(lib().gridadmm_session_branch_costs(self._h, out.ctypes.data_as(_IP)))
        return out[: self.shapes["lt_ij"]]

    def step_counters(self):
        """(TRON its 4-var, 6-var [reference accounting], executed steps 4-var, 6-var)."""
        out = (ctypes.c_longlong * 4)()
        _check(lib().gridadmm_session_step_counters(self._h, out))
        return tuple(out)

    def counters(self):
        """(TRON iterations of all branch solves, of the rate-limited ones)."""
        t = ctypes.c_longlong()
        s = ctypes.c_longlong()
        _check(lib().gridadmm_session_counters(self._h, ctypes.byref(t), ctypes.byref(s)))
        return t.value, s.value

    def close(self):
        if getattr(self, "_h", None):
            lib().gridadmm_session_free(self._h)
            self._h = None

    __del__ = close


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().gridadmm_nccl_unique_id(buf))
    return buf.raw


def device_count() -> int:
    return lib().gridadmm_device_count()


def probe_tron_qp(H, g, lo, hi, x0, tile: int = 1):
    """Batched device TRON on dense box QPs; tile=1 lane mode, tile=4/8/32 tile modes."""
    count, n = g.shape
    x = np.ascontiguousarray(x0, dtype=np.float64).copy()
    status = np.zeros(count, dtype=np.int32)
    its = np.zeros(count, dtype=np.int32)
    args = [np.ascontiguousarray(a, dtype=np.float64) for a in (H, g, lo, hi)]
    _check(lib().gridadmm_probe_tron_qp(count, n, *[_dp(a) for a in args], _dp(x),
                                        status.ctypes.data_as(_IP), its.ctypes.data_as(_IP),
                                        tile))
    return x, status, its


def fp64_peak(device: int = 0):
    """(DMUL+DADD TFLOP/s, DFMA TFLOP/s) measured on the device."""
    a, b = _D(), _D()
    _check(lib().gridadmm_probe_fp64_peak(device, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def probe_sincos(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.zeros_like(x)
    c = np.zeros_like(x)
    _check(lib().gridadmm_probe_sincos(x.size, _dp(x), _dp(s), _dp(c)))
    return s, c
