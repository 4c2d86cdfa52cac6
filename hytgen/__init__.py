"""Seeded synthetic INPUT generators shared by the oracle side and the CUDA side.

This package holds none of HyTGraph's arithmetic (no cost model, no relaxation,
no hub sort).  It only produces CSR graphs in the paper's input format (CSR with
u64 offsets and u32 neighbour ids) and the SSSP weights
(SURVEY.md C19).  Both the oracle tests and the CUDA path consume its output; it
imports neither of them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhytgen.so")
_SRC = os.path.join(_HERE, "hytgen.c")


def build(force: bool = False) -> str:
    """Compile libhytgen.so with gcc (no GPU needed)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread",
                               "-o", _SO, _SRC])
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        u64, u32p, u64p, dbl = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double
        lib.hytgen_rmat_edges.argtypes = [ctypes.c_int, u64, u64, dbl, dbl, dbl, u64, u32p, u32p]
        lib.hytgen_rmat_csr.argtypes = [ctypes.c_int, u64, u64, dbl, dbl, dbl, u64, ctypes.c_int, u64p, u32p]
        lib.hytgen_csr_from_edges.argtypes = [u64, u64, u32p, u32p, ctypes.c_int, u64p, u32p]
        lib.hytgen_weights.argtypes = [u64, u64p, u32p, u64, u32p]
        lib.hytgen_degree_stats.argtypes = [u64, u64p] + [ctypes.POINTER(ctypes.c_uint64)] * 4
        lib.hytgen_degree_stats.restype = None
        i32 = ctypes.c_int
        lib.hytgen_rmat_degrees.argtypes = [i32, u64, u64, dbl, dbl, dbl, u64, i32, u64, u64, u32p, u32p]
        lib.hytgen_rmat_rows.argtypes = [i32, u64, u64, dbl, dbl, dbl, u64, i32, u32p, u64, u64p, u32p, u64]
        lib.hytgen_weights_rows.argtypes = [u64, u32p, u64p, u32p, u64, u32p]
        _lib = lib
    return _lib


def aligned_empty(n: int, dtype, align: int = 4096) -> np.ndarray:
    """Page-aligned numpy array (so the CUDA side may cudaHostRegister it).  Large
    arrays are private anonymous mappings advised for transparent huge pages, which
    makes page-locking them ~5x cheaper (tools/pin_bench.cu)."""
    import mmap
    dtype = np.dtype(dtype)
    nbytes = max(1, n) * dtype.itemsize
    if nbytes >= (64 << 20) and hasattr(mmap, "MADV_HUGEPAGE"):
        huge = 2 << 20
        m = mmap.mmap(-1, (nbytes + huge - 1) // huge * huge, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        m.madvise(mmap.MADV_HUGEPAGE)
        return np.frombuffer(m, dtype=dtype, count=n)
    raw = np.empty(nbytes + align, dtype=np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off:off + n * dtype.itemsize].view(dtype)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class Graph:
    """CSR in original (generator) ids. w is None for unweighted graphs."""
    V: int
    off: np.ndarray  # u64[V+1]
    nbr: np.ndarray  # u32[E]
    w: np.ndarray | None = None
    name: str = ""
    symmetric: bool = False

    @property
    def E(self) -> int:
        return int(self.off[-1])

    def degree_stats(self) -> dict:
        vals = [ctypes.c_uint64() for _ in range(4)]
        _L().hytgen_degree_stats(self.V, _p(self.off), *[ctypes.byref(v) for v in vals])
        lt8, lt32, zero, mx = (v.value for v in vals)
        return {"V": self.V, "E": self.E, "pct_deg_lt8": 100.0 * lt8 / max(1, self.V),
                "pct_deg_lt32": 100.0 * lt32 / max(1, self.V), "pct_deg0": 100.0 * zero / max(1, self.V),
                "max_deg": mx}


def rmat_edges(scale: int, V: int, E: int, abc=(0.57, 0.19, 0.19), seed: int = 1):
    src = np.empty(E, dtype=np.uint32)
    dst = np.empty(E, dtype=np.uint32)
    rc = _L().hytgen_rmat_edges(scale, V, E, abc[0], abc[1], abc[2], seed, _p(src), _p(dst))
    if rc != 0:
        raise ValueError(f"hytgen_rmat_edges rc={rc}")
    return src, dst


def rmat_csr(scale: int, V: int, E: int, abc=(0.57, 0.19, 0.19), seed: int = 1,
             symmetric: bool = False, weighted: bool = False, weight_seed: int | None = None,
             name: str = "") -> Graph:
    stored = E * (2 if symmetric else 1)
    off = aligned_empty(V + 1, np.uint64)
    nbr = aligned_empty(stored, np.uint32)
    rc = _L().hytgen_rmat_csr(scale, V, E, abc[0], abc[1], abc[2], seed, int(symmetric), _p(off), _p(nbr))
    if rc != 0:
        raise ValueError(f"hytgen_rmat_csr rc={rc}")
    g = Graph(V=V, off=off, nbr=nbr, name=name, symmetric=symmetric)
    if weighted:
        g.w = weights(g, seed if weight_seed is None else weight_seed)
    return g


def csr_from_edges(V: int, src, dst, symmetric: bool = False, weighted: bool = False,
                   weights_list=None, weight_seed: int = 7, name: str = "") -> Graph:
    """Crafted graphs. If weights_list is given it must align with (src,dst) and the graph
    must be directed; rows are sorted by dst, weights permuted accordingly."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    M = len(src)
    stored = M * (2 if symmetric else 1)
    off = aligned_empty(V + 1, np.uint64)
    nbr = aligned_empty(stored, np.uint32)
    if weights_list is not None:
        assert not symmetric
        order = np.lexsort((dst, src))
        src_s, dst_s = src[order], dst[order]
        w = aligned_empty(M, np.uint32)
        w[:] = np.asarray(weights_list, dtype=np.uint32)[order]
        off[:] = np.concatenate([[0], np.cumsum(np.bincount(src_s, minlength=V))]).astype(np.uint64)
        nbr[:] = dst_s
        return Graph(V=V, off=off, nbr=nbr, w=w, name=name, symmetric=False)
    rc = _L().hytgen_csr_from_edges(V, M, _p(src), _p(dst), int(symmetric), _p(off), _p(nbr))
    if rc != 0:
        raise ValueError(f"hytgen_csr_from_edges rc={rc}")
    g = Graph(V=V, off=off, nbr=nbr, name=name, symmetric=symmetric)
    if weighted:
        g.w = weights(g, weight_seed)
    return g


def weights(g: Graph, seed: int) -> np.ndarray:
    w = aligned_empty(g.E, np.uint32)
    _L().hytgen_weights(g.V, _p(g.off), _p(g.nbr), seed, _p(w))
    return w


# Workload recipes.  scale/V/E/abc/seed/symmetric.
CONFIGS = {
    "r16": dict(scale=16, V=65_536, E=1 << 20, abc=(0.57, 0.19, 0.19), seed=16, symmetric=False),
    "tw": dict(scale=26, V=41_700_000, E=1_470_000_000, abc=(0.48, 0.21, 0.21), seed=2, symmetric=False),
    "fr": dict(scale=26, V=65_600_000, E=1_806_000_000, abc=(0.45, 0.22, 0.22), seed=3, symmetric=True),
    "uk": dict(scale=27, V=105_900_000, E=3_740_000_000, abc=(0.57, 0.19, 0.19), seed=4, symmetric=False),
    "r30": dict(scale=30, V=1 << 30, E=1 << 34, abc=(0.57, 0.19, 0.19), seed=5, symmetric=True),
}


def scaled(name: str, shift: int) -> dict:
    """The same recipe shrunk by 2**shift in V and E (same edge factor and skew)."""
    c = dict(CONFIGS[name])
    c["scale"] = max(1, c["scale"] - shift)
    c["V"] = max(2, c["V"] >> shift)
    c["E"] = max(1, c["E"] >> shift)
    return c


def make(name: str, shift: int = 0, weighted: bool = False) -> Graph:
    c = scaled(name, shift) if shift else dict(CONFIGS[name])
    return rmat_csr(c["scale"], c["V"], c["E"], c["abc"], c["seed"], c["symmetric"],
                    weighted=weighted, weight_seed=c["seed"] + 1000,
                    name=name if not shift else f"{name}>>{shift}")


# ---------------------------------------------------------------- per-rank shards
# (SURVEY §7.2 #6): no process ever holds the whole graph.  Every edge is a pure
# function of its index, so a rank counts the degrees of its slice of edge indices
# (the caller sums the slices over ranks) and regenerates every edge to keep the
# rows of the vertices it owns.

def recipe(name: str, shift: int = 0) -> dict:
    return scaled(name, shift) if shift else dict(CONFIGS[name])


def rmat_degrees(c: dict, e0: int, e1: int, out_deg=None, in_deg=None):
    """Add the stored out-/in-degrees of edges [e0, e1) of recipe c into u32[V] arrays."""
    V = c["V"]
    if out_deg is None:
        out_deg = np.zeros(V, dtype=np.uint32)
    if in_deg is None:
        in_deg = np.zeros(V, dtype=np.uint32)
    rc = _L().hytgen_rmat_degrees(c["scale"], V, c["E"], *c["abc"], c["seed"], int(c["symmetric"]), e0, e1,
                                  _p(out_deg), _p(in_deg))
    if rc != 0:
        raise ValueError(f"hytgen_rmat_degrees rc={rc}")
    return out_deg, in_deg


def rmat_rows(c: dict, rows: np.ndarray, out_deg: np.ndarray, weighted: bool = False):
    """The CSR rows of original vertices `rows` (in that order) of recipe c: returns
    (off_local u64[n+1], nbr u32[...], w u32[...] | None), each row sorted ascending
    exactly as in rmat_csr's full CSR; neighbour ids stay original."""
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    n = len(rows)
    slot = np.full(c["V"], 0xFFFFFFFF, dtype=np.uint32)
    slot[rows] = np.arange(n, dtype=np.uint32)
    cap = int(out_deg[rows].astype(np.uint64).sum())
    off = aligned_empty(n + 1, np.uint64)
    nbr = aligned_empty(cap, np.uint32)
    rc = _L().hytgen_rmat_rows(c["scale"], c["V"], c["E"], *c["abc"], c["seed"], int(c["symmetric"]),
                               _p(slot), n, _p(off), _p(nbr), cap)
    if rc != 0:
        raise ValueError(f"hytgen_rmat_rows rc={rc}")
    w = None
    if weighted:
        w = aligned_empty(cap, np.uint32)
        _L().hytgen_weights_rows(n, _p(rows), _p(off), _p(nbr), c["seed"] + 1000, _p(w))
    return off, nbr, w
