"""GPU parity for the SURVEY §8f #4 extensions, against the CPU oracle:

- pull (bottom-up, topology-driven) iterations for BFS and CC on symmetric graphs
  whose edges are device-resident, with the per-iteration push/pull switch
  (direction = 1, Beamer's rule) and pull forced in every iteration (direction = 2);
  the long-list slice kernel is exercised by lowering pull_heavy;
- the ImpTM-UM comparison engine (engine_mode = um: edges in managed memory,
  ReadMostly, budget enforced by a balloon), for all four algorithms.

BFS / SSSP / CC bit-exact, PR within 1e-4 relative (BASELINE.json north_star)."""
import functools

import numpy as np
import pytest

import hytgen
import oracle

pytestmark = pytest.mark.gpu

PR_TOL = 1e-4


def sym_graphs():
    out = []
    for i, (scale, ef, abc) in enumerate([(10, 4, (0.57, 0.19, 0.19)), (12, 8, (0.45, 0.22, 0.22)),
                                           (14, 16, (0.57, 0.19, 0.19)), (13, 3, (0.25, 0.25, 0.25)),
                                           (16, 12, (0.57, 0.19, 0.19))]):
        V = (1 << scale) - 37 * i
        out.append((f"sym{i}_s{scale}", scale, V, V * ef // 2, abc, 500 + i))
    return out


SYMS = sym_graphs()


@functools.lru_cache(maxsize=None)
def sym_graph(i):
    name, scale, V, E, abc, seed = SYMS[i]
    return hytgen.rmat_csr(scale, V, E, abc, seed, symmetric=True, weighted=True, weight_seed=seed + 1, name=name)


def crafted_sym():
    gs = []
    V = 5000   # a star (one list far above pull_heavy) plus a path hanging off a leaf
    src = [0] * (V - 1) + list(range(1, V - 1))
    dst = list(range(1, V)) + list(range(2, V))
    gs.append(hytgen.csr_from_edges(V, src, dst, symmetric=True, name="star_path"))
    gs.append(hytgen.csr_from_edges(40, [0, 1, 2, 10, 11, 20], [1, 2, 3, 11, 12, 20], symmetric=True,
                                    name="components"))
    gs.append(hytgen.csr_from_edges(7, [], [], symmetric=True, name="no_edges"))
    return gs


CRAFTED = crafted_sym()


def graph_of(key):
    kind, i = key
    return sym_graph(i) if kind == "rmat" else CRAFTED[i]


@functools.lru_cache(maxsize=None)
def expected(key, algo):
    g = graph_of(key)
    if algo == "bfs":
        return oracle.bfs(g.off, g.nbr, 0)
    if algo == "sssp":
        return oracle.sssp(g.off, g.nbr, g.w, 0)
    if algo == "cc":
        return oracle.cc(g.off, g.nbr)
    r, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-12)
    return r


def run(hyt, g, algo, symmetric=True, budget=0, **params):
    G = hyt.Graph(device=0, budget=budget)
    try:
        G.load(g.off, g.nbr, g.w, symmetric=symmetric)
        for k, v in params.items():
            G.set(k, v)
        G.run(algo, 0)
        return G.values(), G.stats(), G.iter_log()
    finally:
        G.close()


KEYS = [("rmat", i) for i in range(len(SYMS))] + [("crafted", i) for i in range(len(CRAFTED))]


@pytest.mark.parametrize("key", KEYS, ids=lambda k: f"{k[0]}{k[1]}")
@pytest.mark.parametrize("algo", ["bfs", "cc"])
@pytest.mark.parametrize("direction", [0, 1, 2])
@pytest.mark.parametrize("heavy", [32, 1024])
def test_pull_parity(hyt, key, algo, direction, heavy):
    g = graph_of(key)
    got, st, log = run(hyt, g, algo, engine_mode="resident", direction=direction, pull_heavy=heavy)
    assert np.array_equal(got, expected(key, algo))
    if direction == 0:
        assert st["pull_iters"] == 0
    if direction == 2 and g.E:
        assert st["pull_iters"] == st["iterations"] and all(r["dir"] == 1 for r in log)
    assert st["pull_iters"] == sum(r["dir"] for r in log)


def test_pull_switches_both_ways(hyt):
    """Beamer's rule on a power-law graph: push at the start, pull in the dense middle
    iterations, push again at the tail."""
    key = ("rmat", 4)
    g = graph_of(key)
    got, st, log = run(hyt, g, "bfs", engine_mode="resident", direction=1)
    assert np.array_equal(got, expected(key, "bfs"))
    dirs = [r["dir"] for r in log]
    assert dirs[0] == 0 and 1 in dirs, dirs
    assert st["pull_iters"] < st["iterations"]


def test_pull_needs_symmetric_flag_and_residency(hyt):
    key = ("rmat", 2)
    g = graph_of(key)
    # not declared symmetric: push only
    got, st, _ = run(hyt, g, "bfs", symmetric=False, engine_mode="resident", direction=2)
    assert np.array_equal(got, expected(key, "bfs")) and st["pull_iters"] == 0
    # out-of-core (hybrid, small partitions): push only
    got, st, _ = run(hyt, g, "cc", engine_mode="hybrid", partition_bytes=4096, direction=2)
    assert np.array_equal(got, expected(key, "cc")) and st["pull_iters"] == 0
    # SSSP / PR never pull
    got, st, _ = run(hyt, g, "sssp", engine_mode="resident", direction=2)
    assert np.array_equal(got, expected(key, "sssp")) and st["pull_iters"] == 0


def test_pull_with_full_edge_cache(hyt):
    """The hybrid with an edge cache that holds every partition is resident: pull applies."""
    key = ("rmat", 2)
    g = graph_of(key)
    for algo in ("bfs", "cc"):
        got, st, _ = run(hyt, g, algo, engine_mode="hybrid", edge_cache=1, direction=2, budget=256 << 20)
        assert np.array_equal(got, expected(key, algo))
        assert st["pull_iters"] == st["iterations"] > 0


@pytest.mark.parametrize("key", [("rmat", 0), ("rmat", 2), ("rmat", 4), ("crafted", 0)], ids=str)
@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
@pytest.mark.parametrize("budget", [0, 64 << 20])
def test_um_parity(hyt, key, algo, budget):
    g = graph_of(key)
    if algo == "sssp" and g.w is None:
        pytest.skip("unweighted")
    got, st, _ = run(hyt, g, algo, budget=budget, engine_mode="um", direction=0)
    want = expected(key, algo)
    if algo == "pr":
        rel = np.abs(got.astype(np.float64) - want) / want
        assert rel.max() <= PR_TOL
    else:
        assert np.array_equal(got, want)
    assert st["bytes_filter"] == st["bytes_compaction"] == st["bytes_zerocopy"] == 0
    if g.E:
        assert st["parts_resident"] > 0
    if budget:
        assert st["um_balloon_bytes"] > 0
        assert st["device_bytes_peak"] <= budget
    else:
        assert st["um_balloon_bytes"] == 0


def test_um_with_pull(hyt):
    key = ("rmat", 3)
    g = graph_of(key)
    got, st, _ = run(hyt, g, "cc", engine_mode="um", direction=2)
    assert np.array_equal(got, expected(key, "cc")) and st["pull_iters"] == st["iterations"]


def test_um_repeat_runs_and_warm(hyt):
    """Repeated runs on one handle (cold eviction each time, then warm pages)."""
    key = ("rmat", 2)
    g = graph_of(key)
    G = hyt.Graph(device=0, budget=64 << 20)
    try:
        G.load(g.off, g.nbr, g.w, symmetric=True)
        G.set("engine_mode", "um")
        for cold in (1, 1, 0, 0):
            G.set("um_cold", cold)
            G.run("sssp", 0)
            assert np.array_equal(G.values(), expected(key, "sssp"))
    finally:
        G.close()


@pytest.fixture(scope="module")
def fr_small():
    return hytgen.make("fr", shift=3)          # FR-shaped recipe at 1/8 scale, symmetrised


@pytest.mark.parametrize("algo", ["bfs", "cc"])
def test_pull_fr_scale(hyt, fr_small, algo):
    """FR-shaped graph at 1/8 scale (8.2M V, 451M stored edges), resident, push/pull
    switching against the oracle, bit-exact, and pull must pay off."""
    g = fr_small
    want = oracle.bfs(g.off, g.nbr, 0) if algo == "bfs" else oracle.cc(g.off, g.nbr)
    G = hyt.Graph(device=0)
    try:
        G.load(g.off, g.nbr, None, symmetric=True)
        G.set("engine_mode", "resident")
        ms = {}
        for d in (0, 1):
            G.set("direction", d)
            G.run(algo, 0)
            G.run(algo, 0)
            st = G.stats()
            assert np.array_equal(G.values(), want), d
            assert (st["pull_iters"] > 0) == (d == 1)
            ms[d] = st["time_ns"]
    finally:
        G.close()
    if algo == "bfs":    # bottom-up steps skip most edges (measured 5.5x on the full FR shape)
        assert ms[1] < ms[0], ms


def test_symmetric_flag_checked_at_load(hyt):
    """A directed graph declared symmetric fails the in-degree = out-degree check."""
    g = hytgen.rmat_csr(10, 1024, 8192, seed=77)          # directed
    G = hyt.Graph(device=0)
    try:
        with pytest.raises(hyt.HytError) as ei:
            G.load(g.off, g.nbr, symmetric=True)
        assert ei.value.code == hyt.HYT_EINVAL and "HYT_SYMMETRIC" in str(ei.value)
    finally:
        G.close()
