"""GPU parity of the multi-rank path on one device.

`world` handles, one per thread, join an in-process group (hyt_init_dist_local):
the same vertex-range split, per-iteration reductions (min for BFS/SSSP/CC, sum for
PR deltas and ranks), owner-side frontier merge and global termination as a NCCL
job, with the reductions carried through host memory.  Every rank's gathered
result must equal the oracle's: bit-exact for BFS/SSSP/CC, 1e-4 relative for PR."""
import itertools
import threading

import numpy as np
import pytest

from test_gpu_parity import CRAFTED, assert_pr_close, expected, gkey_graph, src_of, symmetric_version

pytestmark = pytest.mark.gpu

_group = itertools.count(1000)


def run_ranks(hyt, g, algo, world, engine="hybrid", part=4096, budget=0, symmetric=False, per_rank=None, **kw):
    key = next(_group)
    out, err = [None] * world, [None] * world

    def body(r):
        G = None
        try:
            G = hyt.Graph(device=0, budget=budget)
            G.init_dist_local(r, world, key)
            G.load(g.off, g.nbr, g.w, symmetric=symmetric)
            G.set("engine_mode", engine)
            G.set("partition_bytes", part)
            for k, v in kw.items():
                G.set(k, v)
            for k, v in (per_rank or {}).items():
                G.set(k, v[r])
            G.run(algo, src_of(g) if algo in ("bfs", "sssp") else 0)
            out[r] = (G.values(), G.stats())
        except Exception as e:          # noqa: BLE001 -- re-raised in the main thread
            err[r] = e
        finally:
            if G is not None:
                G.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    assert all(o is not None for o in out)
    return out


def check(gkey, algo, outs):
    want = expected(gkey, algo)
    for vals, _ in outs:
        if algo == "pr":
            assert_pr_close(vals, want)
        else:
            assert np.array_equal(vals, want)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("engine", ["hybrid", "filter", "compaction", "zerocopy", "resident"])
@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
@pytest.mark.parametrize("gi", [4, 9])
def test_multirank_engines(hyt, world, engine, algo, gi):
    gkey = ("rmat", gi)
    g = symmetric_version(gkey) if algo == "cc" else gkey_graph(gkey)
    outs = run_ranks(hyt, g, algo, world, engine=engine)
    check(gkey, algo, outs)
    # the ranks agree on the iteration count (global termination)
    assert len({st["iterations"] for _, st in outs}) == 1


@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
@pytest.mark.parametrize("ci", range(len(CRAFTED)))
def test_multirank_crafted(hyt, algo, ci):
    """Crafted graphs at world 4: stars whose hub holds more than E/world edges
    (ranks without vertices), chains, isolated vertices, the empty edge set."""
    gkey = ("crafted", ci)
    g = symmetric_version(gkey) if algo == "cc" else gkey_graph(gkey)
    outs = run_ranks(hyt, g, algo, 4)
    check(gkey, algo, outs)


@pytest.mark.parametrize("algo", ["bfs", "sssp", "pr"])
def test_multirank_budget_and_cache(hyt, algo):
    """Per-rank device budget with the partial edge cache: each rank caches a prefix
    of its own partitions."""
    gkey = ("rmat", 13)
    g = gkey_graph(gkey)
    d1 = 4          # ids, or SSSP records packed into 4 bytes (pack_weights)
    outs = run_ranks(hyt, g, algo, 2, part=4096, edge_cache=1, edge_cache_bytes=g.E * d1 // 4)
    check(gkey, algo, outs)
    assert sum(st["parts_resident"] for _, st in outs) > 0


@pytest.mark.parametrize("exchange", [0, 1, 2])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
@pytest.mark.parametrize("engine", ["hybrid", "zerocopy"])
def test_multirank_exchange_modes(hyt, exchange, world, algo, engine):
    """the dense V-entry all-reduce (0), the per-iteration choice (1)
    and the sparse pair all-gather whenever it fits (2) give the oracle's results."""
    gkey = ("rmat", 9)
    g = symmetric_version(gkey) if algo == "cc" else gkey_graph(gkey)
    outs = run_ranks(hyt, g, algo, world, engine=engine, exchange=exchange)
    check(gkey, algo, outs)
    for _, st in outs:
        assert st["exch_sparse"] + st["exch_dense"] == st["iterations"]
        if exchange == 0:
            assert st["exch_sparse"] == 0
        if exchange == 2:
            assert st["exch_sparse"] > 0


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
@pytest.mark.parametrize("engine", ["hybrid", "filter", "compaction", "zerocopy", "resident"])
@pytest.mark.parametrize("gi", [4, 9])
def test_multirank_peer_push(hyt, world, algo, engine, gi):
    """exchange = 3: the relax kernels write remote destinations straight into their
    owners' arrays (fused push, no exchange collective); oracle's results."""
    gkey = ("rmat", gi)
    g = symmetric_version(gkey) if algo == "cc" else gkey_graph(gkey)
    outs = run_ranks(hyt, g, algo, world, engine=engine, exchange=3)
    check(gkey, algo, outs)
    for _, st in outs:
        assert st["exch_peer"] == st["iterations"] > 0
        assert st["exch_sparse"] == st["exch_dense"] == 0


@pytest.mark.parametrize("ci", range(len(CRAFTED)))
@pytest.mark.parametrize("algo", ["bfs", "sssp", "pr"])
def test_multirank_peer_push_crafted(hyt, ci, algo):
    gkey = ("crafted", ci)
    g = gkey_graph(gkey)
    outs = run_ranks(hyt, g, algo, 2, engine="hybrid", exchange=3)
    check(gkey, algo, outs)


def test_multirank_peer_push_repeat_runs(hyt):
    """Several runs on the same handles: bitmaps swap parity across runs, pointers are
    re-published, cached contexts are reused."""
    gkey = ("rmat", 4)
    g = gkey_graph(gkey)
    seq = ["sssp", "pr", "bfs", "sssp", "bfs"]
    world, key = 3, next(_group)
    res, err = [[None] * len(seq) for _ in range(world)], [None] * world

    def body(r):
        G = None
        try:
            G = hyt.Graph(device=0)
            G.init_dist_local(r, world, key)
            G.load(g.off, g.nbr, g.w)
            G.set("partition_bytes", 4096)
            G.set("exchange", 3)
            for j, algo in enumerate(seq):
                G.run(algo, src_of(g) if algo in ("bfs", "sssp") else 0)
                res[r][j] = G.values()
        except Exception as e:          # noqa: BLE001
            err[r] = e
        finally:
            if G is not None:
                G.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for j, algo in enumerate(seq):
        want = expected(gkey, algo)
        for r in range(world):
            if algo == "pr":
                assert_pr_close(res[r][j], want)
            else:
                assert np.array_equal(res[r][j], want), (algo, j, r)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("direction", [1, 2])
@pytest.mark.parametrize("exchange", [0, 1, 3])
@pytest.mark.parametrize("gi", [3, 4, 8, 11])
def test_multirank_pull_bfs(hyt, world, direction, exchange, gi):
    """Pull (bottom-up) BFS across ranks: the frontier is the OR of every rank's own
    words; levels stay bit-exact with every exchange mode."""
    gkey = ("rmat", gi)
    g = symmetric_version(gkey)
    want = oracle_bfs_sym(gkey)
    outs = run_ranks(hyt, g, "bfs", world, engine="resident", symmetric=True, direction=direction,
                     exchange=exchange, pull_heavy=64)
    for vals, st in outs:
        assert np.array_equal(vals, want)
        assert st["pull_iters"] > 0
        if direction == 2:
            assert st["pull_iters"] == st["iterations"]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("direction", [1, 2])
@pytest.mark.parametrize("exchange", [0, 1, 2, 3])
@pytest.mark.parametrize("gi", [3, 4, 8])
def test_multirank_pull_cc(hyt, world, direction, exchange, gi):
    """Pull CC across ranks reads the neighbours' labels from the local full-length copy,
    which the dense / sparse exchanges keep current; with the peer push (3) it stays push."""
    gkey = ("rmat", gi)
    g = symmetric_version(gkey)
    outs = run_ranks(hyt, g, "cc", world, engine="resident", symmetric=True, direction=direction,
                     exchange=exchange, pull_heavy=64)
    check(gkey, "cc", outs)
    for _, st in outs:
        if exchange == 3:
            assert st["pull_iters"] == 0
        else:
            assert st["pull_iters"] > 0
            if direction == 2:
                assert st["pull_iters"] == st["iterations"]


def test_multirank_pull_needs_every_rank_resident(hyt):
    """An edge cache that holds every partition on some ranks only: no rank pulls."""
    gkey = ("rmat", 7)
    g = symmetric_version(gkey)
    want = oracle_bfs_sym(gkey)
    # rank 0 caches everything it owns, rank 1 a quarter of its edges
    outs = run_ranks(hyt, g, "bfs", 2, engine="hybrid", symmetric=True, direction=2, edge_cache=1,
                     per_rank={"edge_cache_bytes": [0, g.E * 4 // 8]})
    for vals, st in outs:
        assert np.array_equal(vals, want)
        assert st["pull_iters"] == 0
    assert outs[0][1]["parts_resident"] > 0
    # both cache everything: pull
    outs = run_ranks(hyt, g, "bfs", 2, engine="hybrid", symmetric=True, direction=2, edge_cache=1)
    for vals, st in outs:
        assert np.array_equal(vals, want)
        assert st["pull_iters"] == st["iterations"] > 0


_bfs_sym_cache = {}


def oracle_bfs_sym(gkey):
    if gkey not in _bfs_sym_cache:
        import oracle
        g = symmetric_version(gkey)
        _bfs_sym_cache[gkey] = oracle.bfs(g.off, g.nbr, src_of(g))
    return _bfs_sym_cache[gkey]


def run_nccl_world1(hyt, g, algo, engine="hybrid", part=4096, symmetric=False, **kw):
    """One handle on a one-rank NCCL communicator (hyt_init_dist at world 1): the
    run takes the multi-rank path -- split, per-iteration NCCL all-reduce / all-gather
    or the CUDA-IPC peer push, owner frontier merge, global termination -- on the
    transport a job uses, where each collective is an identity."""
    import torch  # noqa: F401 -- loads torch's libnccl.so.2, which hyt dlopens
    G = hyt.Graph(device=0)
    try:
        G.init_dist(0, 1, hyt.nccl_unique_id())
        G.load(g.off, g.nbr, g.w, symmetric=symmetric)
        G.set("engine_mode", engine)
        G.set("partition_bytes", part)
        for k, v in kw.items():
            G.set(k, v)
        G.run(algo, src_of(g) if algo in ("bfs", "sssp") else 0)
        return G.values(), G.stats()
    finally:
        G.close()


@pytest.mark.parametrize("exchange", [0, 2, 3])
@pytest.mark.parametrize("engine", ["hybrid", "filter", "compaction", "zerocopy", "resident"])
@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc", "pr"])
def test_nccl_world1(hyt, exchange, engine, algo):
    """The NCCL transport itself (not the in-process group) on the one GPU a test box
    has: dense all-reduce (0), sparse pair all-gather (2), CUDA-IPC peer push (3)."""
    gkey = ("rmat", 9)
    g = symmetric_version(gkey) if algo == "cc" else gkey_graph(gkey)
    vals, st = run_nccl_world1(hyt, g, algo, engine=engine, exchange=exchange)
    check(gkey, algo, [(vals, st)])
    if exchange == 3:
        assert st["exch_peer"] == st["iterations"] > 0
    else:
        assert st["exch_sparse"] + st["exch_dense"] == st["iterations"] > 0
        assert (st["exch_sparse"] > 0) == (exchange == 2)


@pytest.mark.parametrize("direction", [1, 2])
def test_nccl_world1_pull(hyt, direction):
    """Pull BFS across the NCCL path (frontier words all-reduced every pull iteration)."""
    gkey = ("rmat", 9)
    g = symmetric_version(gkey)
    vals, st = run_nccl_world1(hyt, g, "bfs", engine="resident", symmetric=True, direction=direction, exchange=0,
                               pull_heavy=64)
    assert np.array_equal(vals, oracle_bfs_sym(gkey))
    assert st["pull_iters"] > 0
