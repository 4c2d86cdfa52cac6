"""CPU ORACLE for the HyTGraph hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product package (paper_2208_14935_b200) never
imports it and shares no code with it (oracle.c includes only libc).

Every function follows PAPER.md (P:n) in its plain definition or, for the
heuristics (cost model, Algorithm 1, hub sort), step by step in the paper's order.
Pins live in tests/test_oracle_*.py; see DESIGN.md §"Oracle and its pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

INF32 = 0xFFFFFFFF
NONE, F, C, Z = 0, 1, 2, 3


_FLAGS = ["-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """liboracle.so (the Makefile's flags).  ORACLE_LIB=<path> loads another build of
    the same oracle.c instead (bench.py's cpu_baseline compiles one with
    -march=native on the box it runs on)."""
    if os.environ.get("ORACLE_LIB"):
        return os.environ["ORACLE_LIB"]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *_FLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


def build_native(path: str) -> str:
    """The same oracle.c built for the host it runs on (-O3 -march=native), for timing."""
    subprocess.check_call(["gcc", "-O3", "-march=native", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                           "-o", path, _SRC, "-lm"])
    return path


class _CostCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("d1", "d2", "m", "mr", "alpha_num", "alpha_den", "beta_num", "beta_den",
                 "gamma_num", "gamma_den", "k")]


@dataclass
class CostCfg:
    """Cost-model constants.  Thresholds are exact rationals."""
    d1: int = 4
    d2: int = 4
    m: int = 128
    mr: int = 256
    alpha: Fraction = Fraction(4, 5)
    beta: Fraction = Fraction(2, 5)
    gamma: Fraction = Fraction(5, 8)
    k: int = 4

    def c(self) -> _CostCfg:
        return _CostCfg(self.d1, self.d2, self.m, self.mr, self.alpha.numerator, self.alpha.denominator,
                        self.beta.numerator, self.beta.denominator, self.gamma.numerator,
                        self.gamma.denominator, self.k)


_lib = None


def _L():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, vp, i32 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.oracle_bfs.argtypes = [u64, vp, vp, u64, vp]
        L.oracle_sssp.argtypes = [u64, vp, vp, vp, u64, vp]
        L.oracle_cc.argtypes = [u64, vp, vp, vp]
        L.oracle_pr_jacobi.argtypes = [u64, vp, vp, ctypes.c_double, ctypes.c_double, i32, vp, ctypes.POINTER(i32)]
        L.oracle_pr_jacobi_pull.argtypes = [u64, vp, vp, ctypes.c_double, ctypes.c_double, i32, i32, vp,
                                            ctypes.POINTER(i32)]
        L.oracle_pr_delta.argtypes = [u64, vp, vp, ctypes.c_double, ctypes.c_double, vp, ctypes.POINTER(u64)]
        L.oracle_check_bfs.argtypes = [u64, vp, vp, u64, vp]
        L.oracle_check_sssp.argtypes = [u64, vp, vp, vp, u64, vp]
        L.oracle_check_cc.argtypes = [u64, vp, vp, vp]
        L.oracle_pr_residual.argtypes = [u64, vp, vp, ctypes.c_double, vp] + [ctypes.POINTER(ctypes.c_double)] * 3
        L.oracle_hub_sort.argtypes = [u64, vp, vp, u64, u64, vp]
        L.oracle_relabel.argtypes = [u64, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_partition.argtypes = [u64, vp, u64, u64, vp]
        L.oracle_partition.restype = u64
        L.oracle_am.argtypes = [u64, u64, u64]
        L.oracle_am.restype = u64
        cp = ctypes.POINTER(_CostCfg)
        L.oracle_zc_requests.argtypes = [u64, u64, cp]
        L.oracle_zc_requests.restype = u64
        for n in ("oracle_tef", "oracle_nz"):
            getattr(L, n).argtypes = [u64, cp]
            getattr(L, n).restype = u64
        L.oracle_tec.argtypes = [u64, u64, cp]
        L.oracle_tec.restype = u64
        L.oracle_select.argtypes = [u64, u64, u64, u64, cp]
        L.oracle_select.restype = i32
        L.oracle_plan.argtypes = [u64, vp, vp, vp, u64, vp, cp, vp] + [vp] * 7
        L.oracle_select_cal.argtypes = [u64, u64, u64, u64, u64, cp, vp]
        L.oracle_select_cal.restype = i32
        L.oracle_plan.restype = ctypes.c_int64
        L.oracle_combine.argtypes = [u64, vp, u64, vp]
        L.oracle_combine.restype = ctypes.c_int64
        L.oracle_order_units.argtypes = [ctypes.c_int64, vp, vp, vp]
        L.oracle_order_units.restype = None
        _lib = L
    return _lib


def _p(a):
    return 0 if a is None else a.ctypes.data


def _csr(off, nbr):
    off = np.ascontiguousarray(off, dtype=np.uint64)
    nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
    return off, nbr, len(off) - 1


def bfs(off, nbr, src: int) -> np.ndarray:
    off, nbr, V = _csr(off, nbr)
    out = np.empty(V, dtype=np.uint32)
    rc = _L().oracle_bfs(V, _p(off), _p(nbr), src, _p(out))
    if rc:
        raise ValueError(f"oracle_bfs rc={rc}")
    return out


def sssp(off, nbr, w, src: int) -> np.ndarray:
    off, nbr, V = _csr(off, nbr)
    w = np.ascontiguousarray(w, dtype=np.uint32)
    out = np.empty(V, dtype=np.uint32)
    rc = _L().oracle_sssp(V, _p(off), _p(nbr), _p(w), src, _p(out))
    if rc:
        raise ValueError(f"oracle_sssp rc={rc}")
    return out


def cc(off, nbr) -> np.ndarray:
    off, nbr, V = _csr(off, nbr)
    out = np.empty(V, dtype=np.uint32)
    _L().oracle_cc(V, _p(off), _p(nbr), _p(out))
    return out


def pr_jacobi(off, nbr, d: float = 0.85, tol: float = 1e-13, max_iter: int = 100000):
    off, nbr, V = _csr(off, nbr)
    out = np.empty(V, dtype=np.float64)
    it = ctypes.c_int()
    _L().oracle_pr_jacobi(V, _p(off), _p(nbr), d, tol, max_iter, _p(out), ctypes.byref(it))
    return out, it.value


def pr_jacobi_pull(off, nbr, d: float = 0.85, tol: float = 1e-13, max_iter: int = 100000, threads: int = 0):
    """O4a in pull form over a transposed CSR, vertex range split over POSIX threads
    (threads = 0: all host cores).  Same map and stopping rule as pr_jacobi; used at
    the large parity sizes where the single-threaded push form takes minutes."""
    off, nbr, V = _csr(off, nbr)
    out = np.empty(V, dtype=np.float64)
    it = ctypes.c_int()
    nt = threads or (os.cpu_count() or 1)
    _L().oracle_pr_jacobi_pull(V, _p(off), _p(nbr), d, tol, max_iter, nt, _p(out), ctypes.byref(it))
    return out, it.value


def pr_delta(off, nbr, d: float = 0.85, eps: float = 1e-12):
    off, nbr, V = _csr(off, nbr)
    out = np.empty(V, dtype=np.float64)
    pops = ctypes.c_uint64()
    _L().oracle_pr_delta(V, _p(off), _p(nbr), d, eps, _p(out), ctypes.byref(pops))
    return out, pops.value


def check_bfs(off, nbr, src, level) -> int:
    off, nbr, V = _csr(off, nbr)
    level = np.ascontiguousarray(level, dtype=np.uint32)
    return _L().oracle_check_bfs(V, _p(off), _p(nbr), src, _p(level))


def check_sssp(off, nbr, w, src, dist) -> int:
    off, nbr, V = _csr(off, nbr)
    w = np.ascontiguousarray(w, dtype=np.uint32)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    return _L().oracle_check_sssp(V, _p(off), _p(nbr), _p(w), src, _p(dist))


def check_cc(off, nbr, label) -> int:
    off, nbr, V = _csr(off, nbr)
    label = np.ascontiguousarray(label, dtype=np.uint32)
    return _L().oracle_check_cc(V, _p(off), _p(nbr), _p(label))


def pr_residual(off, nbr, rank, d: float = 0.85):
    off, nbr, V = _csr(off, nbr)
    rank = np.ascontiguousarray(rank, dtype=np.float32)
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _L().oracle_pr_residual(V, _p(off), _p(nbr), d, _p(rank), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return {"res_l1": a.value, "sum": b.value, "max_rel_res": c.value}


def hub_sort(off, nbr, frac: Fraction = Fraction(8, 100)) -> np.ndarray:
    off, nbr, V = _csr(off, nbr)
    new_id = np.empty(V, dtype=np.uint32)
    _L().oracle_hub_sort(V, _p(off), _p(nbr), frac.numerator, frac.denominator, _p(new_id))
    return new_id


def relabel(off, nbr, w, new_id):
    off, nbr, V = _csr(off, nbr)
    new_id = np.ascontiguousarray(new_id, dtype=np.uint32)
    off2 = np.empty(V + 1, dtype=np.uint64)
    nbr2 = np.empty(len(nbr), dtype=np.uint32)
    w2 = None
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.uint32)
        w2 = np.empty(len(nbr), dtype=np.uint32)
    _L().oracle_relabel(V, _p(off), _p(nbr), _p(w), _p(new_id), _p(off2), _p(nbr2), _p(w2))
    return off2, nbr2, w2


def partition(off, d1: int, target_bytes: int) -> np.ndarray:
    off = np.ascontiguousarray(off, dtype=np.uint64)
    V = len(off) - 1
    bounds = np.empty(V + 2, dtype=np.uint64)
    n = _L().oracle_partition(V, _p(off), d1, target_bytes, _p(bounds))
    return bounds[: n + 1].copy()


def am(start_byte: int, len_bytes: int, m: int = 128) -> int:
    return _L().oracle_am(start_byte, len_bytes, m)


def zc_requests(off_v: int, deg: int, cfg: CostCfg) -> int:
    c = cfg.c()
    return _L().oracle_zc_requests(off_v, deg, ctypes.byref(c))


def tef(t: int, cfg: CostCfg) -> int:
    c = cfg.c()
    return _L().oracle_tef(t, ctypes.byref(c))


def tec(e: int, a: int, cfg: CostCfg) -> int:
    c = cfg.c()
    return _L().oracle_tec(e, a, ctypes.byref(c))


def nz(z: int, cfg: CostCfg) -> int:
    c = cfg.c()
    return _L().oracle_nz(z, ctypes.byref(c))


def select(t: int, e: int, a: int, z: int, cfg: CostCfg) -> int:
    c = cfg.c()
    return _L().oracle_select(t, e, a, z, ctypes.byref(c))


class _Cal(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("cpu_num", "cpu_den", "zr_num", "zs_num", "z_den")]


@dataclass
class Cal:
    """Calibrated constants as exact rationals: link/Thpt_cpt, and the zero-copy
    random-request (zr) and streamed-line (zs) costs in RTT units."""
    cpu: Fraction
    zr: Fraction
    zs: Fraction

    def c(self) -> _Cal:
        den = self.zr.denominator * self.zs.denominator
        return _Cal(self.cpu.numerator, self.cpu.denominator, int(self.zr * den), int(self.zs * den), den)


def select_cal(t: int, e: int, a: int, z: int, r: int, cfg: CostCfg, cal: Cal) -> int:
    c, k = cfg.c(), cal.c()
    return _L().oracle_select_cal(t, e, a, z, r, ctypes.byref(c), ctypes.byref(k))


@dataclass
class Plan:
    t: np.ndarray
    e: np.ndarray
    a: np.ndarray
    z: np.ndarray
    hub: np.ndarray
    p: np.ndarray
    units: list


def plan(off, active, bounds, cfg: CostCfg, din=None, cal: Cal = None) -> Plan:
    off = np.ascontiguousarray(off, dtype=np.uint64)
    V = len(off) - 1
    active = np.ascontiguousarray(active, dtype=np.uint8)
    bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
    N = len(bounds) - 1
    t, e, a, z, hub = (np.empty(N, dtype=np.uint64) for _ in range(5))
    p = np.empty(N, dtype=np.uint8)
    units = np.empty(2 * N + 2, dtype=np.uint64)
    if din is not None:
        din = np.ascontiguousarray(din, dtype=np.uint64)
    c = cfg.c()
    k = cal.c() if cal is not None else None
    nu = _L().oracle_plan(V, _p(off), _p(din), _p(active), N, _p(bounds), ctypes.byref(c),
                          ctypes.byref(k) if k is not None else None,
                          _p(t), _p(e), _p(a), _p(z), _p(hub), _p(p), _p(units))
    return Plan(t, e, a, z, hub, p, [(int(units[2 * j]), int(units[2 * j + 1])) for j in range(nu)])


def combine(p, k: int = 4) -> list:
    p = np.ascontiguousarray(p, dtype=np.uint8)
    units = np.empty(2 * len(p) + 2, dtype=np.uint64)
    nu = _L().oracle_combine(len(p), _p(p), k, _p(units))
    return [(int(units[2 * j]), int(units[2 * j + 1])) for j in range(nu)]


def order_units(units, part_score) -> list:
    nu = len(units)
    u = np.array([x for pr in units for x in pr] or [0], dtype=np.uint64)
    s = np.ascontiguousarray(part_score, dtype=np.float64)
    order = np.empty(max(1, nu), dtype=np.uint32)
    _L().oracle_order_units(nu, _p(u), _p(s), _p(order))
    return order[:nu].tolist()
