"""Multi-GPU host logic on CPU (world size 2, gloo, 127.0.0.1).

The B200 path shards by vertex range: rank r serves the contiguous run of
partitions `hyt_rank_range` gives it, pushes into a full-length copy of the
values, and once per iteration the ranks reduce (min for BFS/SSSP/CC, sum for PR
deltas), the owners add vertices another rank improved to their next frontier,
PR zeroes its non-owned delta entries (they are an outbox), and a sum of the
active counts decides termination (csrc/engine.cu, csrc/dist.cu).

These tests run that exact protocol with torch.distributed/gloo collectives on
CPU tensors, using the library's own rank split, and check the results against
the oracle.  The per-rank relax step here is a plain synchronous push (the GPU's
engines are covered by the -m gpu parity tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hytgen
import oracle
import paper_2208_14935_b200 as hyt

INF = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(symmetric=False):
    return hytgen.rmat_csr(11, 2000, 24000, seed=31, symmetric=symmetric, weighted=True)


def _push_min(g, vals, frontier, algo, lo, hi):
    """one synchronous push from own active vertices into the full-length copy."""
    new = vals.copy()
    improved = np.zeros(g.V, dtype=bool)
    for u in np.nonzero(frontier[lo:hi])[0] + lo:
        for k in range(int(g.off[u]), int(g.off[u + 1])):
            v = int(g.nbr[k])
            cand = vals[u] + (1 if algo == "bfs" else int(g.w[k])) if algo != "cc" else vals[u]
            if cand < new[v]:
                new[v] = cand
                improved[v] = True
    return new, improved


def _worker(rank, world, port, algo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(symmetric=(algo == "cc"))
        rr = hyt.rank_range(g.off, 8 if algo == "sssp" else 4, 4096, world, rank)
        lo, hi = rr["v_lo"], rr["v_hi"]
        V = g.V
        if algo == "pr":
            d = 0.85
            rank_v = np.zeros(V)
            delta = np.zeros(V)
            delta[lo:hi] = 1 - d                       # only owners hold initial residuals
            for _ in range(2000):
                act = np.zeros(V, dtype=bool)
                act[lo:hi] = delta[lo:hi] > 1e-9
                n = torch.tensor([int(act.sum())], dtype=torch.int64)
                dist.all_reduce(n)
                if n.item() == 0:
                    break
                for u in np.nonzero(act)[0]:
                    du = delta[u]
                    delta[u] = 0.0
                    rank_v[u] += du
                    deg = int(g.off[u + 1] - g.off[u])
                    for k in range(int(g.off[u]), int(g.off[u + 1])):
                        delta[int(g.nbr[k])] += d * du / deg
                t = torch.from_numpy(delta)
                dist.all_reduce(t)                    # owners: residual + everyone's pushes
                delta = t.numpy().copy()
                delta[:lo] = 0.0                      # non-owned entries are an outbox again
                delta[hi:] = 0.0
            t = torch.from_numpy(rank_v)
            dist.all_reduce(t)
            q.put((rank, rr, t.numpy()))
            return
        vals = np.full(V, INF, dtype=np.int64)
        if algo == "cc":
            vals = np.arange(V, dtype=np.int64)
            frontier = np.ones(V, dtype=bool)
        else:
            vals[0] = 0
            frontier = np.zeros(V, dtype=bool)
            frontier[0] = True
        for _ in range(10 * V):
            n = torch.tensor([int(frontier[lo:hi].sum())], dtype=torch.int64)
            dist.all_reduce(n)
            if n.item() == 0:
                break
            vals, improved = _push_min(g, vals, frontier, algo, lo, hi)
            snap = vals[lo:hi].copy()
            t = torch.from_numpy(vals)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            vals = t.numpy().copy()
            nxt = np.zeros(V, dtype=bool)
            nxt[lo:hi] = improved[lo:hi] | (vals[lo:hi] < snap)   # owner-side frontier merge
            frontier = nxt
        q.put((rank, rr, vals))
    finally:
        dist.destroy_process_group()


def _run(algo, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, algo, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def test_rank_ranges_tile_and_balance():
    g = hytgen.rmat_csr(14, 16384, 300000, seed=3)
    for world in (1, 2, 4, 8):
        rs = [hyt.rank_range(g.off, 4, 65536, world, r) for r in range(world)]
        assert rs[0]["p_lo"] == 0 and rs[-1]["p_hi"] == rs[0]["num_parts"]
        assert rs[0]["v_lo"] == 0 and rs[-1]["v_hi"] == g.V
        for a, b in zip(rs, rs[1:]):
            assert a["p_hi"] == b["p_lo"] and a["v_hi"] == b["v_lo"]
        off = g.off.astype(np.int64)
        share = [off[r["v_hi"]] - off[r["v_lo"]] for r in rs]
        # each rank within one partition (+ the largest single vertex) of E/world
        slack = 65536 // 4 + int(np.diff(off).max())
        assert max(abs(s - g.E / world) for s in share) <= slack


@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc"])
def test_gloo_min_exchange_matches_oracle(algo):
    out = _run(algo)
    g = _graph(symmetric=(algo == "cc"))
    want = {"bfs": lambda: oracle.bfs(g.off, g.nbr, 0), "sssp": lambda: oracle.sssp(g.off, g.nbr, g.w, 0),
            "cc": lambda: oracle.cc(g.off, g.nbr)}[algo]()
    for rank, rr, vals in out:
        got = np.where(vals >= INF, INF, vals).astype(np.uint32)
        assert np.array_equal(got, want), rank
    assert out[0][1]["v_hi"] == out[1][1]["v_lo"]


def test_gloo_pr_outbox_exchange_matches_oracle():
    out = _run("pr")
    g = _graph()
    want, _ = oracle.pr_jacobi(g.off, g.nbr)
    for rank, rr, r in out:
        assert np.max(np.abs(r - want) / want) < 1e-7


def test_rank_split_independent_of_partitioning():
    """The vertex-range split depends on the offsets only (one pinned edge store per
    rank serves every algorithm and partition size), cuts at the first vertex whose
    offset reaches r*E/world, and no partition crosses a cut."""
    g = hytgen.rmat_csr(13, 8192, 120000, seed=5)
    off = g.off.astype(np.int64)
    for world in (2, 3, 8):
        for r in range(world):
            rs = [hyt.rank_range(g.off, d1, pb, world, r) for d1 in (4, 8) for pb in (4096, 65536, 32 << 20)]
            assert len({(x["v_lo"], x["v_hi"]) for x in rs}) == 1
            lo = rs[0]["v_lo"]
            want = 0 if r == 0 else int(np.searchsorted(off, g.E * r // world, side="left"))
            assert lo == want


def test_rank_split_hub_larger_than_share():
    """A star whose hub holds most edges: ranks past the hub's share own nothing,
    the ranges still tile [0, V)."""
    V = 1000
    src = [0] * 900 + list(range(1, 100))
    dst = list(range(1, 901)) + list(range(2, 101))
    g = hytgen.csr_from_edges(V, src, dst, name="bighub")
    world = 4
    rs = [hyt.rank_range(g.off, 4, 4096, world, r) for r in range(world)]
    assert rs[0]["v_lo"] == 0 and rs[-1]["v_hi"] == V
    for a, b in zip(rs, rs[1:]):
        assert a["v_hi"] == b["v_lo"] and a["p_hi"] == b["p_lo"]
    assert any(x["v_hi"] == x["v_lo"] for x in rs)


# --------------------------------------------------------------------------- exchange = 3
# The fused peer push on CPU: shared-memory tensors stand in for the peer pointers
# (rank r's value array and its two frontier bitmaps, which every rank can write),
# a per-owner lock stands in for the atomics, and gloo gives the barrier after the
# pushes, the termination sum and the final MIN all-reduce.  Bitmaps swap in
# lockstep, so iteration parity picks the owner's "next" bitmap (csrc/engine.cu).

def _peer_worker(rank, world, port, algo, shared, locks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(symmetric=(algo == "cc"))
        rr = [hyt.rank_range(g.off, 8 if algo == "sssp" else 4, 4096, world, r) for r in range(world)]
        lo, hi = rr[rank]["v_lo"], rr[rank]["v_hi"]
        owner = np.zeros(g.V, dtype=np.int64)
        for r in range(world):
            owner[rr[r]["v_lo"]:rr[r]["v_hi"]] = r
        val = [shared[r][0].numpy() for r in range(world)]
        bm = [[shared[r][1].numpy(), shared[r][2].numpy()] for r in range(world)]
        mine = val[rank]
        mine[:] = np.arange(g.V) if algo == "cc" else INF     # init own array (full length)
        if algo != "cc" and lo <= 0 < hi:
            mine[0] = 0
        bm[rank][0][:] = False
        bm[rank][1][:] = False
        bm[rank][0][lo:hi] = True if algo == "cc" else (np.arange(lo, hi) == 0)
        dist.barrier()                                          # publish: initialised before any push
        it = 0
        while True:
            cur, nxt = bm[rank][it & 1], [bm[r][(it + 1) & 1] for r in range(world)]
            n = torch.tensor([int(cur[lo:hi].sum())], dtype=torch.int64)
            dist.all_reduce(n)
            if n.item() == 0:
                break
            for u in np.nonzero(cur[lo:hi])[0] + lo:
                for k in range(int(g.off[u]), int(g.off[u + 1])):
                    v = int(g.nbr[k])
                    cand = mine[u] + (1 if algo == "bfs" else int(g.w[k])) if algo != "cc" else mine[u]
                    o = int(owner[v])
                    with locks[o]:                              # atomicMin on the owner, then its bit
                        if cand < val[o][v]:
                            val[o][v] = cand
                            nxt[o][v] = True
                    if o != rank:
                        mine[v] = min(mine[v], cand)            # local copy: a filter only
            cur[lo:hi] = False                                  # owner clears its consumed bitmap
            dist.barrier()                                      # every push has landed
            it += 1
        t = torch.from_numpy(mine.astype(np.int64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.MIN)                # owners' values everywhere
        q.put((rank, it, t.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo", ["bfs", "sssp", "cc"])
def test_gloo_peer_push_matches_oracle(algo):
    world = 2
    g = _graph(symmetric=(algo == "cc"))
    shared = [(torch.zeros(g.V, dtype=torch.int64).share_memory_(),
               torch.zeros(g.V, dtype=torch.bool).share_memory_(),
               torch.zeros(g.V, dtype=torch.bool).share_memory_()) for _ in range(world)]
    ctx = mp.get_context("spawn")
    locks = [ctx.Lock() for _ in range(world)]
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, algo, shared, locks, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    if algo == "bfs":
        want = oracle.bfs(g.off, g.nbr, 0)
    elif algo == "sssp":
        want = oracle.sssp(g.off, g.nbr, g.w, 0)
    else:
        want = oracle.cc(g.off, g.nbr)
    for _, iters, vals in out:
        assert iters > 0
        assert np.array_equal(vals.astype(np.uint32), want)


# --------------------------------------------------------------------------- multi-rank pull BFS
# The pull iteration's frontier gather on CPU: each rank masks its frontier bitmap to
# its own vertex range and one SUM all-reduce of the 64-bit words yields the OR (the
# ranks' bits are disjoint); each rank then pulls its own unvisited vertices with the
# iteration's level and the usual MIN exchange follows (csrc/engine.cu, csrc/pull.cu).

def _pull_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(symmetric=True)
        rr = hyt.rank_range(g.off, 4, 4096, world, rank)
        lo, hi = rr["v_lo"], rr["v_hi"]
        V, W = g.V, (g.V + 31) // 32
        vals = np.full(V, INF, dtype=np.int64)
        vals[0] = 0
        front = np.zeros(V, dtype=bool)
        front[0] = True
        it, pulls = 0, 0
        while True:
            n = torch.tensor([int(front[lo:hi].sum())], dtype=torch.int64)
            dist.all_reduce(n)
            if n.item() == 0:
                break
            nxt = np.zeros(V, dtype=bool)
            if it % 2 == 1:            # alternate pull / push iterations
                own = np.zeros(V, dtype=bool)
                own[lo:hi] = front[lo:hi]
                words = np.packbits(np.concatenate([own, np.zeros(64 * ((W + 1) // 2) - V, bool)]),
                                    bitorder="little").view(np.int64).copy()
                t = torch.from_numpy(words)
                dist.all_reduce(t)                          # disjoint bits: the sum is the OR
                glob = np.unpackbits(t.numpy().view(np.uint8), bitorder="little")[:V].astype(bool)
                assert np.array_equal(glob, _all_or(front, lo, hi, world, g))
                for v in range(lo, hi):
                    if vals[v] != INF:
                        continue
                    for k in range(int(g.off[v]), int(g.off[v + 1])):
                        if glob[int(g.nbr[k])]:
                            vals[v] = it + 1
                            nxt[v] = True
                            break
                pulls += 1
            else:
                for u in np.nonzero(front[lo:hi])[0] + lo:
                    for k in range(int(g.off[u]), int(g.off[u + 1])):
                        v = int(g.nbr[k])
                        if vals[u] + 1 < vals[v]:
                            vals[v] = vals[u] + 1
                            nxt[v] = True
            snap = vals[lo:hi].copy()
            t = torch.from_numpy(vals)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            vals = t.numpy().copy()
            front = np.zeros(V, dtype=bool)
            front[lo:hi] = nxt[lo:hi] | (vals[lo:hi] < snap)
            it += 1
        q.put((rank, pulls, vals))
    finally:
        dist.destroy_process_group()


def _all_or(front, lo, hi, world, g):
    """every rank's own frontier is needed; here each rank only knows its own, so the
    check gathers them the slow way (all_gather of the boolean vectors)."""
    own = torch.from_numpy(np.where(np.arange(g.V) >= lo, 1, 0) * np.where(np.arange(g.V) < hi, 1, 0) *
                           front.astype(np.int64))
    outs = [torch.zeros_like(own) for _ in range(world)]
    dist.all_gather(outs, own)
    return (sum(o.numpy() for o in outs) > 0)


def test_gloo_pull_bfs_frontier_or_matches_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_pull_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _graph(symmetric=True)
    want = oracle.bfs(g.off, g.nbr, 0)
    for _, pulls, vals in out:
        assert pulls > 0
        assert np.array_equal(vals.astype(np.uint32), want)
