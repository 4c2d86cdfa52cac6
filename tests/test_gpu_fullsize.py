"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration.

TW (configs[1], the bench workload: 41.7M vertices, 1.47B edges, 16 GB budget,
hybrid): SSSP and BFS are compared element-wise with the oracle's Dijkstra and
queue BFS (about a minute of oracle time at this size); PageRank's Jacobi oracle
takes minutes here, so it runs under HYT_FULLSIZE=1 (below) and the default suite
checks properties that hold at any size (O(E) certificates in oracle.c): the SSSP
certificate (dist[src] = 0, no edge can still relax, every
reached vertex has a tight parent), the BFS level witness, and the PageRank
fixed-point residual; plus exact oracle values on a sample of vertices whose
answer the oracle can compute alone (vertices with in-degree 0: rank exactly 1-d;
the source's distance 0 / level 0; unreachable vertices INF).

Element-wise parity against the oracle at reduced scale, in the bench's launch
configuration under oversubscribing budgets: TW at 1/8 (PR per vertex), FR at 1/4
(CC + BFS bit-exact, CC also through the complete certificate), UK at 1/16 (PR per
vertex + SSSP bit-exact).  PR is compared with the pull-form Jacobi oracle (O4a',
threaded), which finishes these sizes in about a minute.  HYT_FULLSIZE=1 runs them
at full size."""
import functools
import os

import numpy as np
import pytest

import hytgen
import oracle

pytestmark = pytest.mark.gpu
INF = oracle.INF32
FULL = os.environ.get("HYT_FULLSIZE") == "1"


@functools.lru_cache(maxsize=1)
def tw():
    return hytgen.make("tw", weighted=True)


@pytest.fixture(scope="module")
def tw_runs(hyt):
    g = tw()
    G = hyt.Graph(device=0, budget=16 << 30)         # bench.py's configuration
    out = {}
    try:
        G.load(g.off, g.nbr, g.w)
        for a in ("sssp", "bfs", "pr"):
            G.run(a, 0)
            out[a] = (G.values(), G.stats())
    finally:
        G.close()
    return out


def test_tw_sssp_certificate(tw_runs):
    g = tw()
    d, st = tw_runs["sssp"]
    assert oracle.check_sssp(g.off, g.nbr, g.w, 0, d) == 0
    assert st["device_bytes_peak"] <= 16 << 30
    assert st["parts_filter"] > 0 and st["parts_zerocopy"] > 0      # hybrid really mixes engines


def test_tw_sssp_bfs_exact_full_size(tw_runs):
    """The bench's own workload and launch configuration, element by element: SSSP
    (packed records) and BFS on all 41.7M vertices equal the oracle's Dijkstra and
    queue BFS bit for bit (about a minute of single-core oracle time)."""
    g = tw()
    d, st = tw_runs["sssp"]
    assert st["record_bytes"] == 4                                   # TW packs: 26-bit ids, 6-bit weights
    assert np.array_equal(d, oracle.sssp(g.off, g.nbr, g.w, 0))
    lv, _ = tw_runs["bfs"]
    assert np.array_equal(lv, oracle.bfs(g.off, g.nbr, 0))


def test_tw_bfs_certificate(tw_runs):
    g = tw()
    lv, _ = tw_runs["bfs"]
    assert oracle.check_bfs(g.off, g.nbr, 0, lv) == 0
    d, _ = tw_runs["sssp"]
    assert np.array_equal(lv == INF, d == INF)                     # same reachable set


def test_tw_pr_residual_and_samples(tw_runs):
    g = tw()
    r, st = tw_runs["pr"]
    res = oracle.pr_residual(g.off, g.nbr, r)
    # truncation at eps = 1e-5 leaves at most eps/(1-d) = 6.7e-5 relative (DESIGN C16)
    assert res["max_rel_res"] < 1e-4, res
    indeg = np.bincount(g.nbr, minlength=g.V)
    zero_in = np.nonzero(indeg == 0)[0]
    assert len(zero_in) > 1000
    sample = zero_in[:: max(1, len(zero_in) // 5000)]
    assert np.max(np.abs(r[sample] - 0.15) / 0.15) < 1e-6          # r = 1-d exactly (no in-flow)


def _scaled_parity(hyt, name, shift, algos, budget):
    """Element-wise parity against the oracle at 1/2**shift of a BASELINE config, in
    bench.py's launch configuration (hybrid, 32 MiB partitions) under a budget that
    oversubscribes the device: BFS/SSSP/CC bit-exact, PR <= 1e-4 relative per vertex
    against the pull-form Jacobi fixed point (oracle O4a', tol 1e-10 absolute)."""
    g = hytgen.make(name, shift=shift, weighted=("sssp" in algos))
    G = hyt.Graph(device=0, budget=budget)
    try:
        G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
        for a in algos:
            G.run(a, 0)
            got = G.values()
            st = G.stats()
            assert st["device_bytes_peak"] <= budget
            assert st["parts_filter"] + st["parts_zerocopy"] + st["parts_compaction"] > 0   # edges from host
            if a == "cc":
                want = oracle.cc(g.off, g.nbr)
                assert np.array_equal(got, want)
                assert oracle.check_cc(g.off, g.nbr, got) == 0
            elif a == "bfs":
                assert np.array_equal(got, oracle.bfs(g.off, g.nbr, 0))
            elif a == "sssp":
                assert np.array_equal(got, oracle.sssp(g.off, g.nbr, g.w, 0))
            else:
                want, _ = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-10)
                rel = np.abs(got.astype(np.float64) - want) / want
                assert rel.max() < 1e-4, (rel.max(), int(rel.argmax()))
    finally:
        G.close()


def test_tw_shift3_pr_elementwise(hyt):
    """TW recipe at 1/8 (5.2M V, 184M edges) under 2 GB (16 GB / 8): PR per vertex."""
    _scaled_parity(hyt, "tw", 0 if FULL else 3, ["pr"], (16 << 30) if FULL else (2 << 30))


def test_fr_shift2_cc_bfs(hyt):
    """FR recipe at 1/4 (16.4M V, 903M stored edges) under 1 GB (3.6 GB of ids:
    oversubscribed): CC and BFS bit-exact, CC also through the complete certificate."""
    _scaled_parity(hyt, "fr", 0 if FULL else 2, ["cc", "bfs"], (4 << 30) if FULL else (1 << 30))


def test_uk_shift4_pr_sssp(hyt):
    """UK recipe at 1/16 (6.6M V, 234M edges) under 512 MB (1.9 GB of SSSP records):
    PR per vertex and SSSP bit-exact."""
    _scaled_parity(hyt, "uk", 0 if FULL else 4, ["pr", "sssp"], (8 << 30) if FULL else (512 << 20))
