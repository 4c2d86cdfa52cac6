"""paper_2208_14935_b200 -- B200-native HyTGraph hot path (arXiv 2208.14935).

A thin ctypes binding over the C ABI in include/hyt.h (libhyt.so, built for
sm_100a).  Every step of the path runs in the library's CUDA kernels; this module
only marshals arguments.  There is no CPU fallback: importing works without a GPU
(the CPU test suite checks the exports), but every call that needs the device
fails loudly with HytError, and a missing libhyt.so raises at import time.

PyTorch is used only for plumbing: an optional device arena (a torch tensor the
library sub-allocates from) and torch.distributed for the NCCL unique-id broadcast.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhyt.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hyt.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

HYT_OK, HYT_EINVAL, HYT_ENOMEM, HYT_ECUDA, HYT_ESTATE, HYT_ENCCL = 0, -1, -2, -3, -4, -5
HYT_BFS, HYT_SSSP, HYT_CC, HYT_PR = 0, 1, 2, 3
ALGOS = {"bfs": HYT_BFS, "sssp": HYT_SSSP, "cc": HYT_CC, "pr": HYT_PR}
HYT_NO_HUBSORT = 1
HYT_SYMMETRIC = 2
HYT_ADOPT_HOST = 4
MODES = {"hybrid": 0, "filter": 1, "compaction": 2, "zerocopy": 3, "resident": 4, "um": 5}
HYT_ENG_NONE, HYT_ENG_F, HYT_ENG_C, HYT_ENG_Z, HYT_ENG_R = 0, 1, 2, 3, 4
TAGS = ["plan", "filter", "compaction", "zerocopy", "resident", "recompute", "copy", "recompute_queue"]
INF32 = 0xFFFFFFFF


class hyt_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "iterations", "time_ns", "edges_relaxed", "edges_reached", "bytes_filter", "bytes_compaction",
        "bytes_zerocopy", "parts_filter", "parts_compaction", "parts_zerocopy", "parts_resident",
        "units_filter", "device_bytes_peak", "num_partitions")] + [
        (n, ctypes.c_double) for n in ("kernel_ms", "copy_ms", "plan_ms", "gather_ms")] + [
        ("kernel_launches", ctypes.c_uint64), ("eng_ms", ctypes.c_double * 8),
        ("eng_launches", ctypes.c_uint64 * 8), ("eng_chunks", ctypes.c_uint64 * 8), ("eng_edges", ctypes.c_uint64 * 8),
        ("cal_link_gbs", ctypes.c_double), ("cal_cpt_gbs", ctypes.c_double), ("cal_zc_req_ns", ctypes.c_double),
        ("cal_zc_line_ns", ctypes.c_double), ("exch_sparse", ctypes.c_uint64), ("exch_dense", ctypes.c_uint64),
        ("exch_bytes", ctypes.c_uint64), ("pull_iters", ctypes.c_uint64), ("um_balloon_bytes", ctypes.c_uint64),
        ("exch_peer", ctypes.c_uint64), ("host_store_bytes", ctypes.c_uint64),
        ("record_bytes", ctypes.c_uint64)]


class hyt_iter(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_uint64), ("active_vertices", ctypes.c_uint64),
                ("active_edges", ctypes.c_uint64), ("parts_f", ctypes.c_uint32), ("parts_c", ctypes.c_uint32),
                ("parts_z", ctypes.c_uint32), ("parts_r", ctypes.c_uint32), ("units_f", ctypes.c_uint32),
                ("dir", ctypes.c_uint32), ("bytes_f", ctypes.c_uint64), ("bytes_c", ctypes.c_uint64),
                ("bytes_z", ctypes.c_uint64), ("ms", ctypes.c_double)]


_vp, _u64, _i32, _u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32
_SIGS = {
    "hyt_init": ([ctypes.POINTER(_vp), _i32], _i32),
    "hyt_set_device_budget": ([_vp, _u64], _i32),
    "hyt_set_device_arena": ([_vp, _vp, _u64], _i32),
    "hyt_load_csr": ([_vp, _u64, _u64, _vp, _vp, _vp, _u32], _i32),
    "hyt_load_shard_begin": ([_vp, _u64, _vp, _vp, _u32, ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                              ctypes.POINTER(_u64)], _i32),
    "hyt_get_shard_rows": ([_vp, _vp, _u64], _i32),
    "hyt_load_shard_rows": ([_vp, _u64, _vp, _vp, _vp], _i32),
    "hyt_set_param": ([_vp, ctypes.c_char_p, ctypes.c_double], _i32),
    "hyt_run": ([_vp, _i32, _u64], _i32),
    "hyt_get_values": ([_vp, _vp, _u64], _i32),
    "hyt_get_stats": ([_vp, ctypes.POINTER(hyt_stats)], _i32),
    "hyt_get_iter_log": ([_vp, _vp, _u64, ctypes.POINTER(_u64)], _i32),
    "hyt_get_perm": ([_vp, _vp, _u64], _i32),
    "hyt_debug_plan": ([_vp, _i32, _vp, ctypes.POINTER(_u64), _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "hyt_combine": ([_vp, _u64, _u64, _vp], ctypes.c_int64),
    "hyt_order_units": ([ctypes.c_int64, _vp, _vp, _vp], _i32),
    "hyt_select_engine": ([_vp, _u64, _u64, _u64, _u64, _u64], _i32),
    "hyt_nccl_unique_id": ([_vp], _i32),
    "hyt_rank_range": ([_vp, _u64, _u64, _u64, _i32, _i32] + [ctypes.POINTER(_u64)] * 4, ctypes.c_int64),
    "hyt_init_dist": ([_vp, _i32, _i32, _vp], _i32),
    "hyt_init_dist_local": ([_vp, _i32, _i32, _u64], _i32),
    "hyt_free": ([_vp], None),
    "hyt_trim_pinned_cache": ([], None),
    "hyt_last_error": ([], ctypes.c_char_p),
    "hyt_version": ([], ctypes.c_char_p),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res
    globals()[_name] = _f          # same names as the C ABI


def declared_symbols() -> list:
    """Every function include/hyt.h declares (used by the CPU export test)."""
    with open(HEADER_PATH) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hyt_[a-z_0-9]+)\s*\(", txt, re.M)))


class HytError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = hyt_last_error().decode(errors="replace")
        super().__init__(f"{where} failed with code {code}: {msg}")
        self.code = code


def check(rc: int, where: str) -> int:
    if rc < 0:
        raise HytError(rc, where)
    return rc


def _ptr(a):
    return None if a is None else a.ctypes.data


class Graph:
    """One handle = one GPU.  Typical use:

        g = Graph(device=0, budget=16 << 30)
        g.load(off, nbr, w)                 # host numpy arrays (caller ids)
        g.run("sssp", 0)
        dist = g.values()                   # u32[V] by caller id
    """

    def __init__(self, device: int = 0, budget: int = 0, arena: str | None = None, **params):
        h = _vp()
        check(hyt_init(ctypes.byref(h), device), "hyt_init")
        self.h = h
        self.V = 0
        self._arena_tensor = None
        if arena == "torch" and budget:
            import torch
            self._arena_tensor = torch.empty(budget, dtype=torch.uint8, device=f"cuda:{device}")
            check(hyt_set_device_arena(h, self._arena_tensor.data_ptr(), budget), "hyt_set_device_arena")
        elif budget:
            check(hyt_set_device_budget(h, budget), "hyt_set_device_budget")
        for k, v in params.items():
            self.set(k, v)

    def set(self, key: str, value) -> None:
        if key == "engine_mode" and isinstance(value, str):
            value = MODES[value]
        if key == "priority" and isinstance(value, str):
            value = {"auto": -1, "none": 0, "hub": 1, "delta": 2}[value]
        check(hyt_set_param(self.h, key.encode(), float(value)), f"hyt_set_param({key})")

    def init_dist(self, rank: int, world: int, uid: bytes) -> None:
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(hyt_init_dist(self.h, rank, world, buf), "hyt_init_dist")

    def init_dist_local(self, rank: int, world: int, group: int) -> None:
        """Join an in-process group (one thread per rank; testing the multi-rank path on one GPU)."""
        check(hyt_init_dist_local(self.h, rank, world, group), "hyt_init_dist_local")

    @staticmethod
    def _flags(hubsort: bool, symmetric: bool, adopt: bool) -> int:
        return ((0 if hubsort else HYT_NO_HUBSORT) | (HYT_SYMMETRIC if symmetric else 0) |
                (HYT_ADOPT_HOST if adopt else 0))

    def load(self, off, nbr, w=None, hubsort: bool = True, symmetric: bool = False, adopt: bool = False) -> None:
        off = np.ascontiguousarray(off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        if w is not None:
            w = np.ascontiguousarray(w, dtype=np.uint32)
        V = len(off) - 1
        E = int(off[-1]) if V >= 0 else 0
        if adopt:
            self._adopted = nbr             # the library reads it until close()
        check(hyt_load_csr(self.h, V, E, _ptr(off), _ptr(nbr) if E else None, _ptr(w) if w is not None else None,
                           self._flags(hubsort, symmetric, adopt)), "hyt_load_csr")
        self.V = V

    def load_shard_begin(self, out_deg, in_deg, hubsort: bool = True, symmetric: bool = False,
                         adopt: bool = False) -> dict:
        """Two-phase load, step 1 (include/hyt.h): global u32[V] out-/in-degrees by
        caller id -> this rank's internal row range and edge count."""
        out_deg = np.ascontiguousarray(out_deg, dtype=np.uint32)
        in_deg = np.ascontiguousarray(in_deg, dtype=np.uint32)
        lo, hi, ne = _u64(), _u64(), _u64()
        check(hyt_load_shard_begin(self.h, len(out_deg), _ptr(out_deg), _ptr(in_deg),
                                   self._flags(hubsort, symmetric, adopt), ctypes.byref(lo), ctypes.byref(hi),
                                   ctypes.byref(ne)), "hyt_load_shard_begin")
        self.V = len(out_deg)
        return {"row_lo": lo.value, "row_hi": hi.value, "edges": ne.value}

    def shard_rows(self, n: int) -> np.ndarray:
        """Step 2: caller ids of this rank's internal rows, in internal order."""
        out = np.empty(n, dtype=np.uint32)
        check(hyt_get_shard_rows(self.h, _ptr(out) if n else None, n), "hyt_get_shard_rows")
        return out

    def load_shard_rows(self, row_off, nbr, w=None, adopt: bool = False) -> None:
        """Step 3: those rows as a local CSR (caller neighbour ids)."""
        row_off = np.ascontiguousarray(row_off, dtype=np.uint64)
        nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        if w is not None:
            w = np.ascontiguousarray(w, dtype=np.uint32)
        if adopt:
            self._adopted = nbr
        check(hyt_load_shard_rows(self.h, len(row_off) - 1, _ptr(row_off), _ptr(nbr) if len(nbr) else None,
                                  _ptr(w) if w is not None else None), "hyt_load_shard_rows")

    def run(self, algo, source: int = 0) -> None:
        a = ALGOS[algo] if isinstance(algo, str) else int(algo)
        check(hyt_run(self.h, a, source), "hyt_run")
        self._algo = a

    def values(self) -> np.ndarray:
        out = np.empty(self.V, dtype=np.float32 if self._algo == HYT_PR else np.uint32)
        check(hyt_get_values(self.h, _ptr(out), self.V), "hyt_get_values")
        return out

    def values_into(self, out: np.ndarray) -> np.ndarray:
        check(hyt_get_values(self.h, _ptr(out), self.V), "hyt_get_values")
        return out

    def stats(self) -> dict:
        s = hyt_stats()
        check(hyt_get_stats(self.h, ctypes.byref(s)), "hyt_get_stats")
        out = {}
        for n, _ in hyt_stats._fields_:
            v = getattr(s, n)
            out[n] = list(v) if n.startswith("eng_") else v
        return out

    def iter_log(self) -> list:
        n = _u64()
        check(hyt_get_iter_log(self.h, None, 0, ctypes.byref(n)), "hyt_get_iter_log")
        rows = (hyt_iter * max(1, n.value))()
        check(hyt_get_iter_log(self.h, ctypes.cast(rows, _vp), n.value, ctypes.byref(n)), "hyt_get_iter_log")
        return [{f: getattr(rows[i], f) for f, _ in hyt_iter._fields_} for i in range(n.value)]

    def perm(self) -> np.ndarray:
        out = np.empty(self.V, dtype=np.uint32)
        check(hyt_get_perm(self.h, _ptr(out), self.V), "hyt_get_perm")
        return out

    def debug_plan(self, algo, active: np.ndarray) -> dict:
        a = ALGOS[algo] if isinstance(algo, str) else int(algo)
        active = np.ascontiguousarray(active, dtype=np.uint8)
        n = _u64()
        check(hyt_debug_plan(self.h, a, _ptr(active), ctypes.byref(n), None, None, None, None, None, None),
              "hyt_debug_plan")
        N = n.value
        b = np.empty(N + 1, dtype=np.uint64)
        t, e, av, z = (np.empty(N, dtype=np.uint64) for _ in range(4))
        p = np.empty(N, dtype=np.uint8)
        check(hyt_debug_plan(self.h, a, _ptr(active), ctypes.byref(n), _ptr(b), _ptr(t), _ptr(e), _ptr(av),
                             _ptr(z), _ptr(p)), "hyt_debug_plan")
        return {"bounds": b, "t": t, "e": e, "a": av, "z": z, "p": p}

    def close(self) -> None:
        if getattr(self, "h", None):
            hyt_free(self.h)
            self.h = None
        self._arena_tensor = None
        self._adopted = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def combine(p, k: int = 4) -> list:
    p = np.ascontiguousarray(p, dtype=np.uint8)
    units = np.empty(2 * len(p) + 2, dtype=np.uint64)
    n = check(hyt_combine(_ptr(p) if len(p) else None, len(p), k, _ptr(units)), "hyt_combine")
    return [(int(units[2 * j]), int(units[2 * j + 1])) for j in range(n)]


def order_units(units, part_score) -> list:
    """The scheduler's unit order (host routine, no GPU)."""
    nu = len(units)
    u = np.array([x for pr in units for x in pr] or [0], dtype=np.uint64)
    s = np.ascontiguousarray(part_score, dtype=np.float64)
    order = np.empty(max(1, nu), dtype=np.uint32)
    check(hyt_order_units(nu, _ptr(u), _ptr(s), _ptr(order)), "hyt_order_units")
    return order[:nu].tolist()


def select_engine(t: int, e: int, a: int, z: int, d1: int) -> int:
    return check(hyt_select_engine(None, t, e, a, z, d1), "hyt_select_engine")


def rank_range(off, d1: int, partition_bytes: int, world: int, rank: int) -> dict:
    """The library's vertex-range split for `rank` of `world` (host only)."""
    off = np.ascontiguousarray(off, dtype=np.uint64)
    vals = [_u64() for _ in range(4)]
    n = check(hyt_rank_range(_ptr(off), len(off) - 1, d1, partition_bytes, world, rank,
                             *[ctypes.byref(v) for v in vals]), "hyt_rank_range")
    return {"num_parts": n, "p_lo": vals[0].value, "p_hi": vals[1].value, "v_lo": vals[2].value,
            "v_hi": vals[3].value}


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(hyt_nccl_unique_id(buf), "hyt_nccl_unique_id")
    return buf.raw
