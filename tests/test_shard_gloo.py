"""The two-phase shard load's protocol on CPU (world size 2, gloo, 127.0.0.1).

In a multi-GPU job no process holds the whole graph (BASELINE configs[4]):
  1. each rank counts the degrees of its slice of edge indices (hytgen's
     counter-based generator) and the ranks all-reduce the O(V) vectors;
  2. every rank derives the same hub order from those vectors, and
     the library's rank split (hyt_rank_range) on the permuted offsets names the
     rows it serves;
  3. each rank regenerates exactly those rows.
The GPU library's own plan phase is covered by tests/test_gpu_shard.py (its
permutation equals the full load's); here the hub order is the oracle's, so the
test pins the protocol and the generator against the full CSR on CPU: the
summed degrees, the permutation, the bounds and every generated row must equal
what a single process holding the whole graph computes."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hytgen
import oracle
import paper_2208_14935_b200 as hyt

RECIPE = ("r30", 16)     # RMAT-30 recipe at 1/65536 scale: 16384 V, 262144 undirected edges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = hytgen.recipe(*RECIPE)
        E = c["E"]
        od, idg = hytgen.rmat_degrees(c, E * rank // world, E * (rank + 1) // world)
        t = torch.from_numpy(np.stack([od, idg]).astype(np.int64))
        dist.all_reduce(t)                                   # O(V) per rank
        od = t[0].numpy().astype(np.uint32)
        idg = t[1].numpy().astype(np.uint32)
        # the hub order from degrees alone: a graph with these degrees (row content
        # is irrelevant to H(v) = D_o D_i) -- build a stand-in CSR with the right
        # out-degrees whose in-degrees are idg, via the oracle on (off, fake nbr)
        off = np.zeros(c["V"] + 1, dtype=np.uint64)
        off[1:] = np.cumsum(od.astype(np.uint64))
        fake = np.repeat(np.arange(c["V"], dtype=np.uint32), idg.astype(np.int64))
        new_id = oracle.hub_sort(off, fake)
        old_of = np.empty_like(new_id)
        old_of[new_id] = np.arange(c["V"], dtype=np.uint32)
        off_new = np.zeros(c["V"] + 1, dtype=np.uint64)
        off_new[1:] = np.cumsum(od[old_of].astype(np.uint64))
        rr = hyt.rank_range(off_new, 4, 1 << 16, world, rank)
        rows = old_of[rr["v_lo"]:rr["v_hi"]]
        loff, lnbr, lw = hytgen.rmat_rows(c, rows, od, weighted=True)
        q.put((rank, od, idg, new_id, rr, rows, loff, lnbr, lw))
    finally:
        dist.destroy_process_group()


def test_gloo_shard_load_reproduces_full_load():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = hytgen.make(*RECIPE, weighted=True)
    deg = np.diff(g.off.astype(np.int64))
    indeg = np.bincount(g.nbr, minlength=g.V)
    full_perm = oracle.hub_sort(g.off, g.nbr)
    off2, _, _ = oracle.relabel(g.off, g.nbr, g.w, full_perm)
    covered = 0
    for rank, od, idg, new_id, rr, rows, loff, lnbr, lw in res:
        assert np.array_equal(od, deg) and np.array_equal(idg, indeg)
        assert np.array_equal(new_id, full_perm)             # same hub order as one process
        assert rr == hyt.rank_range(off2, 4, 1 << 16, world, rank)
        for i, u in enumerate(rows):                         # every row as in the full CSR
            a, b = int(g.off[u]), int(g.off[u + 1])
            assert np.array_equal(lnbr[loff[i]:loff[i + 1]], g.nbr[a:b])
            assert np.array_equal(lw[loff[i]:loff[i + 1]], g.w[a:b])
        covered += int(loff[-1])
        assert int(loff[-1]) < 0.75 * g.E                    # each rank holds a share, not E
    assert covered == g.E
