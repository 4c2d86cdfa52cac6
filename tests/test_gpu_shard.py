"""GPU tests of the two-phase (shard) load and HYT_ADOPT_HOST (include/hyt.h).

No process holds the whole graph: each rank counts the degrees of its slice of
edge indices, the slices are summed (here in the test; torch.distributed in a
job), the library hub-sorts from the O(V) degree vectors and names the rows the
rank serves, and the rank regenerates exactly those rows with the counter-based
generator (hytgen.rmat_rows).  The results must equal the oracle's on the same
graph, and the permutation must equal the full load's."""
import itertools
import threading

import numpy as np
import pytest

import hytgen
import oracle

pytestmark = pytest.mark.gpu
INF = oracle.INF32
_group = itertools.count(5000)


def degrees(c, world=3):
    """Global degrees as the sum of `world` per-rank slices (what ranks all-reduce)."""
    od = np.zeros(c["V"], dtype=np.uint32)
    idg = np.zeros(c["V"], dtype=np.uint32)
    for r in range(world):
        o, i = hytgen.rmat_degrees(c, c["E"] * r // world, c["E"] * (r + 1) // world)
        od += o
        idg += i
    return od, idg


def shard_load(hyt, G, c, od, idg, weighted, **kw):
    info = G.load_shard_begin(od, idg, symmetric=c["symmetric"], **kw)
    rows = G.shard_rows(info["row_hi"] - info["row_lo"])
    off, nbr, w = hytgen.rmat_rows(c, rows, od, weighted=weighted)
    assert int(off[-1]) == info["edges"]
    G.load_shard_rows(off, nbr, w, adopt=kw.get("adopt", False))
    return info, rows


@pytest.mark.parametrize("name,shift", [("tw", 13), ("r30", 15)])
def test_shard_load_world1_equals_full_load(hyt, name, shift):
    c = hytgen.recipe(name, shift)
    g = hytgen.make(name, shift, weighted=True)
    od, idg = degrees(c)
    assert np.array_equal(od, np.diff(g.off.astype(np.int64)))
    F = hyt.Graph(device=0)
    S = hyt.Graph(device=0)
    try:
        F.load(g.off, g.nbr, g.w, symmetric=g.symmetric)
        info, rows = shard_load(hyt, S, c, od, idg, True)
        assert info["row_lo"] == 0 and info["row_hi"] == g.V and info["edges"] == g.E
        perm = F.perm()
        assert np.array_equal(S.perm(), perm)
        assert np.array_equal(perm[rows], np.arange(g.V, dtype=np.uint32))   # rows = old_of
        for algo in ("bfs", "sssp", "pr"):
            for G in (F, S):
                G.set("partition_bytes", 1 << 16)
                G.run(algo, 0)
            a, b = F.values(), S.values()
            if algo == "pr":
                want, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-12)
                assert np.max(np.abs(b - want) / want) < 1e-4
            else:
                assert np.array_equal(a, b)
        assert S.stats()["host_store_bytes"] == F.stats()["host_store_bytes"] > 0
    finally:
        F.close()
        S.close()


def _ranks(hyt, c, od, idg, world, algo, weighted, budget=0, engine="hybrid", part=1 << 20):
    key = next(_group)
    out, err = [None] * world, [None] * world

    def body(r):
        G = None
        try:
            G = hyt.Graph(device=0, budget=budget)
            G.init_dist_local(r, world, key)
            info, rows = shard_load(hyt, G, c, od, idg, weighted)
            G.set("engine_mode", engine)
            G.set("partition_bytes", part)
            G.run(algo, 0)
            out[r] = (G.values(), G.stats(), info)
        except Exception as e:          # noqa: BLE001 -- re-raised below
            err[r] = e
        finally:
            if G is not None:
                G.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    for e in err:
        if e is not None:
            raise e
    return out


def test_shard_load_world4_r30_shift6_certificates(hyt):
    """RMAT-30 recipe at 1/64 scale (16.8M V, 268M undirected edges -> 537M stored),
    4 in-process ranks each loading only its own rows: BFS and SSSP certificates on
    the full graph, every rank gathering all V values, and each rank's pinned store
    about 1/4 of the graph."""
    c = hytgen.recipe("r30", 6)
    od, idg = degrees(c, world=4)
    E = int(od.astype(np.uint64).sum())
    g = hytgen.make("r30", 6, weighted=True)       # checker side only
    for algo in ("bfs", "sssp"):
        outs = _ranks(hyt, c, od, idg, 4, algo, weighted=True, budget=6 << 30)
        vals = outs[0][0]
        for v, _, _ in outs[1:]:
            assert np.array_equal(v, vals)
        if algo == "bfs":
            assert oracle.check_bfs(g.off, g.nbr, 0, vals) == 0
        else:
            assert oracle.check_sssp(g.off, g.nbr, g.w, 0, vals) == 0
        edges = [info["edges"] for _, _, info in outs]
        assert sum(edges) == E
        for (_, st, info) in outs:
            # ids (4 B) + packed records (8 B) of about E/4 edges, not of E
            assert st["host_store_bytes"] <= 12 * (info["edges"] + 64) + 256
            assert info["edges"] < 0.4 * E


def test_adopt_host_ids(hyt):
    """HYT_ADOPT_HOST + HYT_NO_HUBSORT: the caller's id array is the store (no
    library copy of the ids); results equal the oracle's."""
    g = hytgen.make("tw", 12, weighted=False)
    G = hyt.Graph(device=0)
    try:
        G.load(g.off, g.nbr, hubsort=False, adopt=True)
        G.set("partition_bytes", 1 << 16)
        G.run("bfs", 0)
        assert np.array_equal(G.values(), oracle.bfs(g.off, g.nbr, 0))
        assert G.stats()["host_store_bytes"] == 0
        G.run("pr")
        want, _ = oracle.pr_jacobi(g.off, g.nbr, tol=1e-12)
        assert np.max(np.abs(G.values() - want) / want) < 1e-4
        for mode in ("zerocopy", "compaction", "filter"):
            G.set("engine_mode", mode)
            G.run("bfs", 0)
            assert np.array_equal(G.values(), oracle.bfs(g.off, g.nbr, 0)), mode
    finally:
        G.close()


def test_shard_errors(hyt):
    c = hytgen.recipe("tw", 14)
    od, idg = degrees(c, world=1)
    G = hyt.Graph(device=0)
    try:
        with pytest.raises(hyt.HytError):                 # rows before begin
            G.load_shard_rows(np.zeros(1, np.uint64), np.zeros(0, np.uint32))
        bad = idg.copy()
        bad[0] += 1
        with pytest.raises(hyt.HytError):                 # degree sums differ
            G.load_shard_begin(od, bad)
    finally:
        G.close()
    G = hyt.Graph(device=0)
    try:
        with pytest.raises(hyt.HytError):                 # adopt needs no hub sort
            G.load_shard_begin(od, idg, adopt=True)
    finally:
        G.close()
    G = hyt.Graph(device=0)
    try:
        info = G.load_shard_begin(od, idg)
        rows = G.shard_rows(info["row_hi"] - info["row_lo"])
        off, nbr, _ = hytgen.rmat_rows(c, rows, od)
        wrong = off.copy()
        k = int(np.nonzero(np.diff(off.astype(np.int64)) > 0)[0][0])
        wrong[k + 1] -= 1                                 # a row one edge short
        with pytest.raises(hyt.HytError):
            G.load_shard_rows(wrong, nbr)
        G.load_shard_rows(off, nbr)                       # the right rows still load
        G.run("bfs", 0)
    finally:
        G.close()
