"""ctypes wrapper over oracle/liboracle_f2m.so — the CPU restatement of the reference path.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg as the parity checker; the product package never imports it.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class _Cfg(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int), ("eta", ctypes.c_double), ("eps", ctypes.c_double),
                ("max_sweeps", ctypes.c_int), ("mode", ctypes.c_int), ("update", ctypes.c_int),
                ("init", ctypes.c_int)]


class _Rep(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("sweeps", ctypes.c_int),
                ("final_max_abs_delta", ctypes.c_double), ("dual_value", ctypes.c_double)]


class _RunCfg(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int), ("engine", _Cfg), ("tol", ctypes.c_double),
                ("gap_tol", ctypes.c_double), ("max_restarts", ctypes.c_int),
                ("perturb_scale", ctypes.c_double), ("seed", ctypes.c_uint64)]


class _Outcome(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("gap", ctypes.c_double),
                ("feasible", ctypes.c_int), ("restarts", ctypes.c_int), ("convergence", _Rep)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle_f2m.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", _HERE])
        L = ctypes.CDLL(path)
        L.orc_generate_instance.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_double, _f64p]
        L.orc_distance.argtypes = [_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_distance.restype = ctypes.c_double
        pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_int))
        pd = ctypes.POINTER(ctypes.POINTER(ctypes.c_double))
        for fn in (L.orc_build_knn, L.orc_knn_scan):
            fn.argtypes = [ctypes.c_int, _f64p, ctypes.c_int, ctypes.c_int, pp, pp, pd]
            fn.restype = ctypes.c_int64
        L.orc_free.argtypes = [ctypes.c_void_p]
        L.orc_csr.argtypes = [ctypes.c_int, ctypes.c_int64, _i32p, _i32p, _f64p,
                              np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS"), _i32p]
        L.orc_csr.restype = ctypes.c_double
        g = [ctypes.c_int, ctypes.c_int64, _i32p, _i32p, _f64p]
        L.orc_initial_state.argtypes = g + [ctypes.POINTER(_Cfg), _f64p]
        for fn in (L.orc_jacobi_sweep, L.orc_gauss_seidel_sweep):
            fn.argtypes = g + [ctypes.POINTER(_Cfg), _f64p, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)]
        L.orc_dual_objective.argtypes = g + [_f64p, ctypes.c_int]
        L.orc_dual_objective.restype = ctypes.c_double
        L.orc_solve_duals.argtypes = g + [ctypes.c_double, ctypes.POINTER(_Cfg), ctypes.c_int,
                                          _f64p, ctypes.POINTER(_Rep)]
        L.orc_classify.argtypes = [ctypes.c_int64, _i32p, _i32p, _f64p, _f64p, ctypes.c_double,
                                   _u8p]
        L.orc_extract.argtypes = g + [_f64p, ctypes.c_double, _f64p,
                                      ctypes.POINTER(ctypes.c_double)]
        L.orc_verify.argtypes = g + [_f64p, ctypes.c_double, _f64p, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_double)]
        L.orc_full_solve_graph.argtypes = g + [ctypes.POINTER(_RunCfg), _f64p, _f64p,
                                               ctypes.POINTER(_Outcome)]
        _LIB = L
    return _LIB


@dataclass
class Graph:
    n: int
    eu: np.ndarray
    ev: np.ndarray
    cost: np.ndarray

    @property
    def m(self):
        return int(self.eu.shape[0])

    def args(self):
        return (self.n, self.m, self.eu, self.ev, self.cost)

    def mean_cost(self) -> float:
        off = np.zeros(self.n + 1, np.int64)
        ids = np.zeros(max(2 * self.m, 1), np.int32)
        return lib().orc_csr(*self.args(), off, ids)

    def csr(self):
        off = np.zeros(self.n + 1, np.int64)
        ids = np.zeros(max(2 * self.m, 1), np.int32)
        lib().orc_csr(*self.args(), off, ids)
        return off, ids[: 2 * self.m]


def generate_instance(n: int, seed: int, box: float = 1000.0) -> np.ndarray:
    xy = np.zeros(2 * n, np.float64)
    lib().orc_generate_instance(n, seed, box, xy)
    return xy.reshape(n, 2)


def _edges_call(fn, xy, rounded, k) -> Graph:
    xy = np.ascontiguousarray(xy, np.float64).reshape(-1)
    n = xy.shape[0] // 2
    eu = ctypes.POINTER(ctypes.c_int)()
    ev = ctypes.POINTER(ctypes.c_int)()
    c = ctypes.POINTER(ctypes.c_double)()
    m = fn(n, xy, int(rounded), k, ctypes.byref(eu), ctypes.byref(ev), ctypes.byref(c))
    if m < 0:
        raise ValueError("oracle k-NN: bad arguments")
    a = np.ctypeslib.as_array(eu, (m,)).copy() if m else np.zeros(0, np.int32)
    b = np.ctypeslib.as_array(ev, (m,)).copy() if m else np.zeros(0, np.int32)
    w = np.ctypeslib.as_array(c, (m,)).copy() if m else np.zeros(0, np.float64)
    for p in (eu, ev, c):
        lib().orc_free(ctypes.cast(p, ctypes.c_void_p))
    return Graph(n, a.astype(np.int32), b.astype(np.int32), w)


def build_knn_graph(xy, k: int, rounded: bool = False) -> Graph:
    return _edges_call(lib().orc_build_knn, xy, rounded, k)


def knn_graph_scan(xy, k: int, rounded: bool = False) -> Graph:
    return _edges_call(lib().orc_knn_scan, xy, rounded, k)


def from_edges(n, edges) -> Graph:
    """edges: iterable of (u, v, cost); normalized to u < v and sorted (graph.cpp:14-24)."""
    e = sorted(((min(u, v), max(u, v), c) for u, v, c in edges), key=lambda t: (t[0], t[1]))
    return Graph(n, np.array([t[0] for t in e], np.int32), np.array([t[1] for t in e], np.int32),
                 np.array([t[2] for t in e], np.float64))


def _cfg(b=2, eta=0.5, eps=1e-9, max_sweeps=20000, mode="jacobi", update="midpoint",
         init="local-midpoint"):
    return _Cfg(b, eta, eps, max_sweeps, 1 if mode == "gauss-seidel" else 0,
                1 if update == "paper-difference" else 0, 1 if init == "zero" else 0)


def initial_state(g: Graph, **kw) -> np.ndarray:
    lam = np.zeros(g.n, np.float64)
    lib().orc_initial_state(*g.args(), ctypes.byref(_cfg(**kw)), lam)
    return lam


def jacobi_sweep(g: Graph, lam: np.ndarray, **kw):
    mx, dv = ctypes.c_double(), ctypes.c_double()
    rc = lib().orc_jacobi_sweep(*g.args(), ctypes.byref(_cfg(**kw)), lam, ctypes.byref(mx),
                                ctypes.byref(dv))
    if rc:
        raise RuntimeError(f"oracle jacobi_sweep rc={rc}")
    return mx.value, dv.value


def gauss_seidel_sweep(g: Graph, lam: np.ndarray, **kw):
    mx, dv = ctypes.c_double(), ctypes.c_double()
    rc = lib().orc_gauss_seidel_sweep(*g.args(), ctypes.byref(_cfg(**kw)), lam, ctypes.byref(mx),
                                      ctypes.byref(dv))
    if rc:
        raise RuntimeError(f"oracle gauss_seidel_sweep rc={rc}")
    return mx.value, dv.value


def dual_objective(g: Graph, lam: np.ndarray, b: int = 2) -> float:
    return lib().orc_dual_objective(*g.args(), np.ascontiguousarray(lam, np.float64), b)


def solve_duals(g: Graph, initial=None, **kw):
    lam = np.zeros(g.n, np.float64) if initial is None else np.array(initial, np.float64)
    rep = _Rep()
    rc = lib().orc_solve_duals(*g.args(), g.mean_cost(), ctypes.byref(_cfg(**kw)),
                               0 if initial is None else 1, lam, ctypes.byref(rep))
    if rc:
        raise RuntimeError(f"oracle solve_duals rc={rc}")
    return lam, dict(converged=bool(rep.converged), sweeps=rep.sweeps,
                     final_max_abs_delta=rep.final_max_abs_delta, dual_value=rep.dual_value)


def classify(g: Graph, lam, tol):
    lab = np.zeros(max(g.m, 1), np.uint8)
    if lib().orc_classify(g.m, g.eu, g.ev, g.cost, np.ascontiguousarray(lam, np.float64), tol, lab):
        raise ValueError("tol must be > 0")
    return lab[: g.m]


def extract_primal(g: Graph, lam, tol):
    x = np.zeros(max(g.m, 1), np.float64)
    obj = ctypes.c_double()
    rc = lib().orc_extract(*g.args(), np.ascontiguousarray(lam, np.float64), tol, x,
                           ctypes.byref(obj))
    if rc:
        raise RuntimeError(f"oracle extract rc={rc}")
    return x[: g.m], obj.value


def verify(g: Graph, x, objective, lam):
    vv, gap = ctypes.c_int(), ctypes.c_double()
    bad = lib().orc_verify(*g.args(), np.ascontiguousarray(x, np.float64), objective,
                           np.ascontiguousarray(lam, np.float64), ctypes.byref(vv),
                           ctypes.byref(gap))
    return dict(violated=bad, value_violations=vv.value, gap=gap.value,
                feasible=bad == 0 and vv.value == 0)


def full_solve_graph(g: Graph, k=20, eta=0.5, eps=1e-9, max_sweeps=20000, mode="jacobi", tol=0.0,
                     gap_tol=1e-6, max_restarts=5, perturb_scale=1e-7, seed=0):
    rc_ = _RunCfg(k, _cfg(eta=eta, eps=eps, max_sweeps=max_sweeps, mode=mode), tol, gap_tol,
                  max_restarts, perturb_scale, seed)
    x = np.zeros(max(g.m, 1), np.float64)
    lam = np.zeros(g.n, np.float64)
    out = _Outcome()
    rc = lib().orc_full_solve_graph(*g.args(), ctypes.byref(rc_), x, lam, ctypes.byref(out))
    if rc:
        raise RuntimeError(f"oracle full_solve_graph rc={rc}")
    return dict(objective=out.objective, gap=out.gap, feasible=bool(out.feasible),
                restarts=out.restarts, sweeps=out.convergence.sweeps, value=x[: g.m], duals=lam)
