"""Pins of the CPU oracle's algorithms (O1-O4) against things other than itself:
brute force on tiny graphs, scipy / networkx / numpy.linalg, closed forms,
hand-worked examples (tests/golden/hand_graphs.json) and invariants.
CPU only (-m "not gpu")."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse import csgraph

import hytgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = oracle.INF32
D = 0.85


def hand():
    with open(os.path.join(GOLD, "hand_graphs.json")) as f:
        return json.load(f)


def graph_from(V, edges, weighted=False):
    src = [e[0] for e in edges]
    dst = [e[1] for e in edges]
    if weighted:
        return hytgen.csr_from_edges(V, src, dst, weights_list=[e[2] for e in edges])
    return hytgen.csr_from_edges(V, src, dst)


def random_tiny(seed, V=None, p=None, weighted=False, symmetric=False):
    rng = np.random.default_rng(seed)
    V = V or int(rng.integers(2, 40))
    p = p or float(rng.uniform(0.02, 0.3))
    mask = rng.random((V, V)) < p
    src, dst = np.nonzero(mask)
    g = hytgen.csr_from_edges(V, src, dst, symmetric=symmetric)
    if weighted:
        g.w = hytgen.weights(g, seed)
    return g


def dense_adj(g, weights=False):
    """dense V x V matrix (min weight for parallel edges) for brute force."""
    V = g.V
    A = np.full((V, V), np.inf)
    for u in range(V):
        for k in range(int(g.off[u]), int(g.off[u + 1])):
            v = int(g.nbr[k])
            val = float(g.w[k]) if weights else 1.0
            A[u, v] = min(A[u, v], val)
    return A


def floyd_warshall(A):
    V = A.shape[0]
    Dm = A.copy()
    np.fill_diagonal(Dm, np.minimum(np.diag(Dm), 0.0))
    for k in range(V):
        Dm = np.minimum(Dm, Dm[:, k:k + 1] + Dm[k:k + 1, :])
    return Dm


def to_u32(dist_row):
    return np.where(np.isinf(dist_row), INF, dist_row).astype(np.uint32)


def scipy_matrix(g, weights=False):
    E = g.E
    rows = np.repeat(np.arange(g.V), np.diff(g.off.astype(np.int64)))
    data = g.w.astype(np.float64) if weights else np.ones(E)
    cols = g.nbr.astype(np.int64)
    # parallel edges: scipy would SUM duplicates; shortest paths need the MIN weight
    key = rows * g.V + cols
    order = np.lexsort((data, key))
    key, data = key[order], data[order]
    first = np.concatenate([[True], key[1:] != key[:-1]])
    key, data = key[first], data[first]
    return sp.csr_matrix((data, (key // g.V, key % g.V)), shape=(g.V, g.V))


# ---------------------------------------------------------------- BFS (O1)

def test_bfs_hand_two_paths():
    h = hand()["bfs_two_paths"]
    g = graph_from(h["V"], h["edges"])
    assert oracle.bfs(g.off, g.nbr, h["src"]).tolist() == h["level"]


@pytest.mark.parametrize("seed", range(12))
def test_bfs_brute_force_floyd_warshall(seed):
    g = random_tiny(seed)
    src = seed % g.V
    want = to_u32(floyd_warshall(dense_adj(g))[src])
    assert np.array_equal(oracle.bfs(g.off, g.nbr, src), want)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bfs_vs_scipy_rmat(seed):
    g = hytgen.rmat_csr(12, 4096, 40000, seed=seed)
    want = to_u32(csgraph.shortest_path(scipy_matrix(g), unweighted=True, indices=0))
    got = oracle.bfs(g.off, g.nbr, 0)
    assert np.array_equal(got, want)
    assert oracle.check_bfs(g.off, g.nbr, 0, got) == 0


def test_bfs_equals_sssp_with_unit_weights():
    g = hytgen.rmat_csr(11, 2048, 20000, seed=9)
    ones = np.ones(g.E, dtype=np.uint32)
    assert np.array_equal(oracle.bfs(g.off, g.nbr, 0), oracle.sssp(g.off, g.nbr, ones, 0))


def test_bfs_checker_rejects_mutations():
    g = hytgen.rmat_csr(10, 1024, 8000, seed=5)
    lv = oracle.bfs(g.off, g.nbr, 0)
    assert oracle.check_bfs(g.off, g.nbr, 0, lv) == 0
    reached = np.nonzero((lv != INF) & (lv > 0))[0]
    bad = lv.copy(); bad[reached[3]] += 1
    assert oracle.check_bfs(g.off, g.nbr, 0, bad) != 0
    bad = lv.astype(np.int64); bad[reached[3]] -= 1; bad = bad.astype(np.uint32)
    assert oracle.check_bfs(g.off, g.nbr, 0, bad) != 0


# ---------------------------------------------------------------- SSSP (O2)

def test_sssp_hand():
    for key in ("sssp_triangle", "sssp_disconnected"):
        h = hand()[key]
        g = graph_from(h["V"], h["edges"], weighted=True)
        assert oracle.sssp(g.off, g.nbr, g.w, h["src"]).tolist() == h["dist"], key


@pytest.mark.parametrize("seed", range(12))
def test_sssp_brute_force_floyd_warshall(seed):
    g = random_tiny(seed + 100, weighted=True)
    src = seed % g.V
    want = to_u32(floyd_warshall(dense_adj(g, weights=True))[src])
    assert np.array_equal(oracle.sssp(g.off, g.nbr, g.w, src), want)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_sssp_vs_scipy_dijkstra_rmat(seed):
    g = hytgen.rmat_csr(12, 4096, 40000, seed=seed, weighted=True)
    want = to_u32(csgraph.dijkstra(scipy_matrix(g, weights=True), indices=0))
    got = oracle.sssp(g.off, g.nbr, g.w, 0)
    assert np.array_equal(got, want)
    assert oracle.check_sssp(g.off, g.nbr, g.w, 0, got) == 0


def test_sssp_checker_rejects_mutations():
    g = hytgen.rmat_csr(10, 1024, 8000, seed=6, weighted=True)
    d = oracle.sssp(g.off, g.nbr, g.w, 0)
    reached = np.nonzero((d != INF) & (d > 0))[0]
    for delta in (+1, -1):
        bad = d.astype(np.int64); bad[reached[7]] += delta; bad = bad.astype(np.uint32)
        assert oracle.check_sssp(g.off, g.nbr, g.w, 0, bad) != 0


def test_weights_rule_range_and_symmetry():
    g = hytgen.rmat_csr(10, 1024, 8000, seed=6, symmetric=True, weighted=True)
    assert g.w.min() >= 1 and g.w.max() <= 63
    rows = np.repeat(np.arange(g.V), np.diff(g.off.astype(np.int64)))
    wmap = {}
    for u, v, w in zip(rows.tolist(), g.nbr.tolist(), g.w.tolist()):
        wmap[(u, v)] = w
    for (u, v), w in list(wmap.items())[:2000]:
        assert wmap[(v, u)] == w


# ---------------------------------------------------------------- CC (O3)

def test_cc_hand():
    for key in ("cc_two_edges", "cc_path", "cc_single"):
        h = hand()[key]
        src = [e[0] for e in h["edges"]]
        dst = [e[1] for e in h["edges"]]
        g = hytgen.csr_from_edges(h["V"], src, dst, symmetric=True)
        assert oracle.cc(g.off, g.nbr).tolist() == h["label"], key


def min_id_labels_from_scipy(g):
    n, lab = csgraph.connected_components(scipy_matrix(g), directed=False)
    mins = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(mins, lab, np.arange(g.V))
    return mins[lab].astype(np.uint32), n


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_cc_vs_scipy(seed):
    g = hytgen.rmat_csr(12, 4096, 6000, abc=(0.45, 0.22, 0.22), seed=seed, symmetric=True)
    want, ncomp = min_id_labels_from_scipy(g)
    got = oracle.cc(g.off, g.nbr)
    assert np.array_equal(got, want)
    assert oracle.check_cc(g.off, g.nbr, got) == 0
    assert int((got == np.arange(g.V)).sum()) == ncomp       # fixed points = components


@pytest.mark.parametrize("seed", range(6))
def test_cc_brute_force_closure(seed):
    g = random_tiny(seed + 300, p=0.05, symmetric=True)
    A = np.isfinite(dense_adj(g)) | np.eye(g.V, dtype=bool)
    R = A.copy()
    for k in range(g.V):
        R = R | (R[:, k:k + 1] & R[k:k + 1, :])
    want = np.array([np.nonzero(R[v])[0].min() for v in range(g.V)], dtype=np.uint32)
    assert np.array_equal(oracle.cc(g.off, g.nbr), want)


def test_cc_checker_rejects_mutations():
    g = hytgen.rmat_csr(10, 1024, 3000, seed=8, symmetric=True)
    lab = oracle.cc(g.off, g.nbr)
    big = np.bincount(lab).argmax()
    members = np.nonzero(lab == big)[0]
    bad = lab.copy(); bad[members[-1]] = members[-1]
    assert oracle.check_cc(g.off, g.nbr, bad) != 0


def _sym_csr(V, edges):
    adj = [[] for _ in range(V)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)
    off = np.zeros(V + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(x) for x in adj])
    nbr = np.array([v for x in adj for v in sorted(x)], dtype=np.uint32)
    return off, nbr


def test_cc_checker_golden_cases():
    """tests/golden/cc_certificate_cases.json: hand-worked valid / invalid labellings,
    including the merged-components counterexample a local-invariant check accepts."""
    with open(os.path.join(GOLD, "cc_certificate_cases.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        off, nbr = _sym_csr(c["V"], c["edges"])
        lab = np.array(c["labels"], dtype=np.uint32)
        rc = oracle.check_cc(off, nbr, lab)
        assert (rc == 0) == c["valid"], (c["name"], rc)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_cc_checker_rejects_merged_components(seed):
    """Relabel a whole component with a smaller root of ANOTHER component: every
    local invariant (labels equal across edges, label <= v, label is a fixed point)
    still holds, so only the complete certificate can reject it."""
    g = hytgen.rmat_csr(11, 2048, 2500, abc=(0.45, 0.22, 0.22), seed=seed, symmetric=True)
    lab = oracle.cc(g.off, g.nbr)
    assert oracle.check_cc(g.off, g.nbr, lab) == 0
    roots = np.nonzero(lab == np.arange(g.V))[0]
    assert len(roots) >= 2
    bad = lab.copy()
    bad[lab == roots[-1]] = roots[0]
    assert oracle.check_cc(g.off, g.nbr, bad) != 0


# ---------------------------------------------------------------- PageRank (O4)

def pr_dense_solve(g, d=D):
    V = g.V
    P = np.zeros((V, V))
    for u in range(V):
        deg = int(g.off[u + 1] - g.off[u])
        for k in range(int(g.off[u]), int(g.off[u + 1])):
            P[u, int(g.nbr[k])] += 1.0 / deg
    return np.linalg.solve(np.eye(V) - d * P.T, (1 - d) * np.ones(V))


@pytest.mark.parametrize("seed", range(10))
def test_pr_vs_dense_solve(seed):
    g = random_tiny(seed + 500, p=0.12)          # includes dangling vertices
    want = pr_dense_solve(g)
    rj, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-14)
    rd, _ = oracle.pr_delta(g.off, g.nbr, eps=1e-13)
    assert np.max(np.abs(rj - want) / want) < 1e-11
    assert np.max(np.abs(rd - want) / want) < 1e-10


@pytest.mark.parametrize("seed", range(6))
def test_pr_pull_vs_dense_solve(seed):
    """O4a' (pull-form Jacobi over a transposed CSR, threaded) against the linear
    solve directly, on tiny graphs with dangling vertices and duplicate edges."""
    g = random_tiny(seed + 700, p=0.15)
    want = pr_dense_solve(g)
    for nt in (1, 3):
        got, _ = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-14, threads=nt)
        assert np.max(np.abs(got - want) / want) < 1e-11


def test_pr_pull_thread_count_invariant():
    """Each vertex is summed by one thread in in-list order: the result is the same
    bit for bit for any thread count, and equals the push form to rounding."""
    g = hytgen.rmat_csr(13, 8192, 120000, seed=21)
    a, ia = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-12, threads=1)
    b, ib = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-12, threads=7)
    assert ia == ib and np.array_equal(a, b)
    c, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-12)
    assert np.max(np.abs(a - c) / c) < 1e-10


def test_pr_closed_forms():
    # directed cycle -> all 1 (unnormalised fixed point)
    n = 7
    g = hytgen.csr_from_edges(n, list(range(n)), [(i + 1) % n for i in range(n)])
    rj, _ = oracle.pr_jacobi(g.off, g.nbr)
    rd, _ = oracle.pr_delta(g.off, g.nbr)
    assert np.allclose(rj, 1.0, rtol=0, atol=1e-12) and np.allclose(rd, 1.0, atol=1e-10)
    # complete graph (no self loops) -> all 1
    src, dst = zip(*[(i, j) for i in range(6) for j in range(6) if i != j])
    g = hytgen.csr_from_edges(6, src, dst)
    assert np.allclose(oracle.pr_jacobi(g.off, g.nbr)[0], 1.0, atol=1e-12)
    # in-degree-0 vertex -> exactly 1-d; star 0->{1..8}: leaves 1-d + d(1-d)/8
    g = hytgen.csr_from_edges(9, [0] * 8, list(range(1, 9)))
    rj, _ = oracle.pr_jacobi(g.off, g.nbr)
    rd, _ = oracle.pr_delta(g.off, g.nbr)
    for r in (rj, rd):
        assert r[0] == pytest.approx(1 - D, abs=1e-15)
        assert np.allclose(r[1:], (1 - D) + D * (1 - D) / 8, atol=1e-12)
    # two-cycle with d = 0.5: equal ranks, = 1
    h = hand()["pr_two_cycle"]
    g = graph_from(h["V"], h["edges"])
    assert np.allclose(oracle.pr_jacobi(g.off, g.nbr, d=h["d"])[0], h["rank"], atol=1e-12)


def test_pr_vs_networkx_dangling_free():
    import networkx as nx
    # symmetric graph with no isolated vertices -> dangling free
    g = hytgen.rmat_csr(9, 512, 4000, abc=(0.45, 0.22, 0.22), seed=3, symmetric=True)
    deg = np.diff(g.off.astype(np.int64))
    keep = np.nonzero(deg > 0)[0]
    remap = -np.ones(g.V, dtype=np.int64); remap[keep] = np.arange(len(keep))
    rows = np.repeat(np.arange(g.V), deg)
    src, dst = remap[rows], remap[g.nbr.astype(np.int64)]
    g2 = hytgen.csr_from_edges(len(keep), src, dst)
    G = nx.MultiDiGraph()
    G.add_nodes_from(range(g2.V))
    r2 = np.repeat(np.arange(g2.V), np.diff(g2.off.astype(np.int64)))
    G.add_edges_from(zip(r2.tolist(), g2.nbr.tolist()))
    nxr = nx.pagerank(G, alpha=D, tol=1e-14, max_iter=10000)
    want = np.array([nxr[i] for i in range(g2.V)]) * g2.V
    rj, _ = oracle.pr_jacobi(g2.off, g2.nbr)
    assert np.max(np.abs(rj - want) / want) < 1e-8
    assert rj.sum() == pytest.approx(g2.V, rel=1e-12)      # sum r = V on dangling-free graphs


def test_pr_mass_identity_and_truncation_bound():
    g = hytgen.rmat_csr(13, 8192, 120000, seed=11)
    rj, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-13)
    deg = np.diff(g.off.astype(np.int64))
    # sum r - d * sum_{D_o>0} r = (1-d) V
    assert rj.sum() - D * rj[deg > 0].sum() == pytest.approx((1 - D) * g.V, rel=1e-11)
    for eps in (1e-4, 1e-6, 1e-9):
        rd, _ = oracle.pr_delta(g.off, g.nbr, eps=eps)
        gap = (rj - rd) / rj
        assert gap.min() > -1e-11                      # delta-PR never overshoots r*
        assert gap.max() <= eps / (1 - D) * 1.0001     # 0 <= r* - r <= eps/(1-d) r*


def test_pr_residual_checker():
    g = hytgen.rmat_csr(11, 2048, 20000, seed=12)
    rj, _ = oracle.pr_jacobi(g.off, g.nbr)
    res = oracle.pr_residual(g.off, g.nbr, rj.astype(np.float32))
    assert res["max_rel_res"] < 1e-6
    bad = rj.astype(np.float32); bad[5] *= 1.01
    assert oracle.pr_residual(g.off, g.nbr, bad)["max_rel_res"] > 1e-3
