#!/usr/bin/env python
"""bench.py -- HyTGraph hot path on B200: GTEPS and time-to-converge.

Workload (BASELINE.json configs[1]): a Twitter-shaped RMAT graph (41.7M vertices,
1.47B directed edges, u32 weights 1..63), SSSP from vertex 0 and delta-PageRank
(eps 1e-5) on one B200 with the device budget capped at 16 GB and the edges in
pinned host memory (the paper's storage split): every iteration each
partition is served by the engine the section 5.1 cost model picks.

One STEP = hyt_run(SSSP, 0) + hyt_run(PR) to convergence (inputs resident: the CSR
in pinned host memory, offsets/vertex state in HBM).  value = whole-job GTEPS =
(sum of out-degrees of reached vertices for SSSP + E for PR) / (time of both runs)
(SURVEY C24 GTEPS_in).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config tw] [--shift S] [--budget-gb 16] [--algos sssp,pr]

For N > 1 launch with torchrun (one rank per GPU, NCCL): every rank counts the
degrees of its slice of edge indices, the ranks all-reduce them, and each rank
loads only the rows it serves (the two-phase shard load, include/hyt.h), serves its
contiguous range of partitions, and the ranks reduce the pushed values once per
iteration.  Rank 0 prints ONE JSON line.

Besides the contract's keys the line carries (N = 1):
  extras        one timed run per (config, algorithm, engine mode) after a warm-up:
                R16 resident / hybrid with the oracle's time, TW at 16 GB, FR at 4 GB,
                UK at 8 GB, each in hybrid, filter, zero-copy and (not PR) compaction,
                with transfer / edge volume (Table V / VI analogs);
  cpu_baseline  the oracle built -O3 -march=native on this host, on tw>>6 and a
                full-size Dijkstra on TW, with the host's CPU model and cores;
  roofline      the dominant kernel against the HBM copy peak (the contract) and
                against its access pattern's ceiling (profiles/r02_scatter_bench.json);
  kernels / host_link / engine_ms / per_algo  the rest of the breakdown.
--no-extras / --no-cpu-baseline / --no-cpu-full shorten a run.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS and time-to-converge per algo at 1/2/4/8 B200, % HBM/PCIe peak"
L2_NOTE = ("inputs larger than L2: edges live in pinned host memory (5.9 GB of SSSP records packed as "
           "id | w << 26, 5.9 GB ids) and the vertex state (0.5 GB) exceeds the 126 MB L2")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="tw")
    ap.add_argument("--shift", type=int, default=0, help="shrink the workload by 2**shift (debug only)")
    ap.add_argument("--budget-gb", type=float, default=16.0)
    ap.add_argument("--algos", default="sssp,pr")
    ap.add_argument("--engine", default="hybrid")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-full", action="store_true", help="skip the full-size single-core oracle SSSP")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the per-config / per-algorithm / per-engine-mode comparison runs (N=1 only)")
    ap.add_argument("--cpu-shift", type=int, default=6, help="oracle sample = the workload >> cpu_shift")
    ap.add_argument("--json-out", default="")
    ap.add_argument("--detail-out", default="", help="write per-iteration logs + stats of the last step here")
    ap.add_argument("--dist", action="store_true",
                    help="take the multi-rank path even at N = 1 (NCCL communicator, shard load, per-iteration "
                         "exchange; every collective is an identity at world 1)")
    ap.add_argument("--set", action="append", default=[], help="extra library parameter key=value (experiments)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- workload

def workload_desc(config: str, shift: int, algos) -> str:
    import hytgen
    c = hytgen.scaled(config, shift) if shift else hytgen.CONFIGS[config]
    kind = "undirected (symmetrised)" if c["symmetric"] else "directed"
    return (f"{config}" + (f">>{shift}" if shift else "") + f": RMAT {c['V']} V / {c['E']} E {kind}, "
            "u32 weights 1..63; " + "+".join(algos) + " from vertex 0 (PR eps 1e-5)")


def make_graph(config: str, shift: int, weighted: bool):
    import hytgen
    t = time.time()
    g = hytgen.make(config, shift=shift, weighted=weighted)
    return g, time.time() - t


def reached_edges(g, dist) -> int:
    deg = g.deg if isinstance(g, Workload) else np.diff(g.off.astype(np.int64))
    return int(deg[dist != 0xFFFFFFFF].sum())


class Workload:
    """The graph as this rank holds it.  N = 1: the whole CSR (hyt_load_csr).  N > 1:
    the shard load (include/hyt.h) -- each rank counts the degrees of its slice of
    edge indices, the ranks all-reduce the O(V) degree vectors, the library names the
    rows the rank serves and the rank regenerates only those (hytgen.rmat_rows), so
    no process holds the whole graph (BASELINE configs[4])."""

    def __init__(self, config, shift, weighted, world=1, rank=0, local=0, shard=False):
        import hytgen
        t = time.time()
        self.c = hytgen.recipe(config, shift)
        self.weighted, self.world, self.rank = weighted, world, rank
        self.V, self.symmetric = self.c["V"], bool(self.c["symmetric"])
        self.shard = shard
        self.g = None
        self.rows = self.loff = self.lnbr = self.lw = None
        if not self.shard:
            self.g = hytgen.make(config, shift=shift, weighted=weighted)
            self.deg = np.diff(self.g.off.astype(np.int64))
        else:
            import torch
            import torch.distributed as dist
            E = self.c["E"]
            od, idg = hytgen.rmat_degrees(self.c, E * rank // world, E * (rank + 1) // world)
            t2 = torch.from_numpy(np.stack([od, idg]).view(np.int32)).to(f"cuda:{local}")
            dist.all_reduce(t2)                      # degrees < 2^31: int32 sums are exact
            both = t2.cpu().numpy().view(np.uint32)
            self.od, self.idg = np.ascontiguousarray(both[0]), np.ascontiguousarray(both[1])
            self.deg = self.od.astype(np.int64)
        self.E = int(self.deg.sum())
        self.gen_s = time.time() - t

    def load(self, G):
        if not self.shard:
            g = self.g
            G.load(g.off, g.nbr, g.w if self.weighted else None, symmetric=self.symmetric)
            return
        import hytgen
        info = G.load_shard_begin(self.od, self.idg, symmetric=self.symmetric)
        if self.rows is None:                       # first load: generate this rank's rows
            t = time.time()
            self.rows = G.shard_rows(info["row_hi"] - info["row_lo"])
            self.loff, self.lnbr, self.lw = hytgen.rmat_rows(self.c, self.rows, self.od, weighted=self.weighted)
            self.gen_s += time.time() - t
        G.load_shard_rows(self.loff, self.lnbr, self.lw)

    def host_arrays(self):
        if not self.shard:
            return [self.g.off, self.g.nbr, self.g.w if self.weighted else None]
        return [self.loff, self.lnbr, self.lw, self.od, self.idg]

    def degree_stats(self) -> dict:
        d = self.deg
        return {"V": self.V, "E": self.E, "pct_deg_lt8": 100.0 * float((d < 8).mean()),
                "pct_deg_lt32": 100.0 * float((d < 32).mean()), "pct_deg0": 100.0 * float((d == 0).mean()),
                "max_deg": int(d.max()), "load": "shard (per-rank rows)" if self.shard else "full CSR"}


def measured_h2d_gbs(device: int) -> float:
    """Pinned host->device copy bandwidth on this box (host-link roofline denominator)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    gbs = 4 * n / (s.elapsed_time(e) / 1e3) / 1e9
    del h, d
    torch.cuda.empty_cache()
    return gbs


def pin_host(arrays) -> list:
    """cudaHostRegister (portable | mapped | read-only) of host arrays; returns those registered."""
    import torch
    cr = torch.cuda.cudart()
    done = []
    for a in arrays:
        if a is None or a.nbytes == 0:
            continue
        rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 1 | 2 | 8)
        if rc == 0 or str(rc).endswith("success"):
            done.append(a)
    return done


def unpin_host(arrays) -> None:
    import torch
    cr = torch.cuda.cudart()
    for a in arrays:
        cr.cudaHostUnregister(a.ctypes.data)


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


# --------------------------------------------------------------------------- reference arm

def host_cpu() -> dict:
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def use_native_oracle() -> str:
    """Build the oracle for this host (-O3 -march=native) and make `import oracle` load it."""
    import tempfile
    path = os.path.join(tempfile.gettempdir(), f"hyt_oracle_native_{os.getpid()}.so")
    sys.path.insert(0, ROOT)
    import oracle
    oracle.build_native(path)
    os.environ["ORACLE_LIB"] = path
    oracle._lib = None
    return path


def cpu_oracle_full_sssp(g) -> dict:
    """Dijkstra (the oracle as it stands) once on the FULL workload graph, one core."""
    import oracle
    t = time.perf_counter()
    d = oracle.sssp(g.off, g.nbr, g.w, 0)
    dt = time.perf_counter() - t
    e = reached_edges(g, d)
    return {"algo": "sssp", "graph": g.name or "full", "V": g.V, "E": g.E, "seconds": dt, "edges": e,
            "gteps": e / dt / 1e9}


def cpu_oracle_sample(config: str, shift: int, algos, steps: int = 1):
    """The CPU oracle (as it stands) on a bounded sample of the same workload."""
    import oracle
    g, _ = make_graph(config, shift, weighted=True)
    edges = 0
    secs = 0.0
    for _ in range(steps):
        for a in algos:
            t = time.perf_counter()
            if a == "sssp":
                d = oracle.sssp(g.off, g.nbr, g.w, 0)
                dt = time.perf_counter() - t
                edges += reached_edges(g, d)
            elif a == "bfs":
                d = oracle.bfs(g.off, g.nbr, 0)
                dt = time.perf_counter() - t
                edges += reached_edges(g, d)
            else:
                oracle.pr_delta(g.off, g.nbr, eps=1e-5)
                dt = time.perf_counter() - t
                edges += g.E
            secs += dt
    return {"value": edges / secs / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
            "sample": f"{config}>>{shift} ({g.V} V, {g.E} E), {'+'.join(algos)}, single-threaded C oracle "
                      f"(Dijkstra / sequential delta-PR eps 1e-5), {steps} step(s), {secs:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    algos = args.algos.split(",")
    shift = max(args.shift, args.cpu_shift)
    native = use_native_oracle()
    import oracle
    g, _ = make_graph(args.config, shift, weighted=True)
    times = []
    edges_step = 0
    for i in range(args.warmup + args.steps):
        edges = 0
        t0 = time.perf_counter()
        for a in algos:
            if a == "sssp":
                edges += reached_edges(g, oracle.sssp(g.off, g.nbr, g.w, 0))
            elif a == "bfs":
                edges += reached_edges(g, oracle.bfs(g.off, g.nbr, 0))
            else:
                oracle.pr_delta(g.off, g.nbr, eps=1e-5)
                edges += g.E
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            edges_step = edges
    ms = 1e3 * float(np.mean(times))
    val = edges_step / (ms / 1e3) / 1e9
    sample = (f"{args.config}>>{shift} ({g.V} V, {g.E} E) -- bounded sample of the workload; "
              f"single-threaded C oracle (Dijkstra, sequential delta-PR eps 1e-5)")
    line = {"metric": METRIC, "value": val, "unit": "GTEPS", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32+f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_desc(args.config, args.shift, algos), "budget_gb": args.budget_gb,
                       "engine_mode": args.engine, "reference_sample": f"{args.config}>>{shift}"},
            "cpu_baseline": {"value": val, "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample,
                             "host": host_cpu(), "build": f"gcc -O3 -march=native ({os.path.basename(native)})"},
            "e2e": {"value": val, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- per-config comparison

# (config, device budget GB (0 = none), algorithms): BASELINE.json configs[0..3] at one GPU.
# configs[0] (R16) is the fully resident case; it is timed resident and hybrid, with the
# single-core oracle beside it.
EXTRAS = [("r16", 0, ["bfs", "sssp"]), ("tw", 16, ["sssp", "pr"]), ("fr", 4, ["bfs", "cc"]),
          ("uk", 8, ["sssp", "pr"])]


def run_extras(hyt, local: int, tw_graph=None) -> dict:
    """One timed run per (config, algorithm, engine mode): the hybrid against the pure
    explicit (filter, compaction) and implicit (zero-copy) modes of the same build, with
    the host-link transfer volume normalised to the edge volume (Table V / Table VI
    analogs).  Results must agree across modes."""
    import torch
    out = {}
    for name, bgb, algos in EXTRAS:
        t = time.time()
        g = tw_graph if (name == "tw" and tw_graph is not None) else \
            make_graph(name, 0, weighted=("sssp" in algos))[0]
        gen_s = time.time() - t
        G = hyt.Graph(device=local, budget=int(bgb * (1 << 30)))
        small = name == "r16"
        t = time.time()
        G.load(g.off, g.nbr, g.w if "sssp" in algos else None, symmetric=bool(g.symmetric))
        load_s = time.time() - t
        cur = torch.cuda.current_stream()
        res = {}
        for a in algos:
            modes = ["hybrid", "filter", "zerocopy"] + ([] if a == "pr" else ["compaction"])
            if small:
                modes = ["hybrid", "resident"]
            row, ref = {}, None
            G.set("engine_mode", "hybrid")
            G.run(a, 0)        # untimed: run context + this graph's host-gather calibration
            for m in modes:     # the transfer modes share the run context (no rebuild)
                G.set("engine_mode", m)
                if m == "resident":
                    G.run(a, 0)          # untimed: the resident copy of the edges
                torch.cuda.synchronize()
                s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_ev.record(cur)
                G.run(a, 0)
                e_ev.record(cur)
                torch.cuda.synchronize()
                sec = s_ev.elapsed_time(e_ev) / 1e3
                st = G.stats()
                vals = G.values()
                edges = reached_edges(g, vals) if a in ("sssp", "bfs") else g.E
                d1 = 8 if a == "sssp" else 4      # the paper's edge volume: (id, weight) = 8 B for SSSP
                xfer = st["bytes_filter"] + st["bytes_compaction"] + st["bytes_zerocopy"]
                if ref is None:
                    ref, agree = vals, True
                elif a == "pr":
                    agree = bool(np.max(np.abs(vals - ref) / np.maximum(ref, 1e-30)) < 2e-4)
                else:
                    agree = bool(np.array_equal(vals, ref))
                row[m] = {"s": sec, "gteps": edges / sec / 1e9, "iterations": int(st["iterations"]),
                          "xfer_over_edge_volume": xfer / (g.E * d1),
                          "record_bytes": int(st["record_bytes"]),
                          "xfer_over_store_volume": xfer / (g.E * max(1, int(st["record_bytes"]))),
                          "agrees_with_hybrid": agree,
                          "parts_fcz": [int(st["parts_filter"]), int(st["parts_compaction"]),
                                        int(st["parts_zerocopy"])]}
            if small:
                import oracle
                t = time.perf_counter()
                if a == "bfs":
                    want = oracle.bfs(g.off, g.nbr, 0)
                else:
                    want = oracle.sssp(g.off, g.nbr, g.w, 0)
                row["oracle_1core_s"] = time.perf_counter() - t
                row["equals_oracle"] = bool(np.array_equal(ref, want))
            else:
                others = [row[m]["s"] for m in modes if m != "hybrid"]
                row["hybrid_fastest"] = bool(row["hybrid"]["s"] <= min(others))
                row["speedup_vs_best_pure"] = min(others) / row["hybrid"]["s"]
            res[a] = row
        G.close()
        out[name] = {"workload": workload_desc(name, 0, algos), "budget_gb": bgb, "gen_s": gen_s,
                     "load_s": load_s, "algos": res}
        if g is not tw_graph:
            del g
    return out


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2208_14935_b200 as hyt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    multi = world > 1 or args.dist
    if multi:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    algos = args.algos.split(",")
    budget = int(args.budget_gb * (1 << 30))

    # ---- inputs (host), generation not timed ----
    if world > 1:
        os.environ.setdefault("HYTGEN_THREADS", str(max(1, (os.cpu_count() or 8) // world)))
    g = Workload(args.config, args.shift, "sssp" in algos, world, rank, local, shard=multi)
    dstats = g.degree_stats()

    def new_handle():
        G = hyt.Graph(device=local, budget=budget)
        if multi:
            uid = [hyt.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            G.init_dist(rank, world, uid[0])
        G.set("engine_mode", args.engine)
        for kv in args.set:
            k, v = kv.split("=")
            G.set(k, float(v))
        return G

    G = new_handle()
    t = time.time()
    g.load(G)
    load_s = time.time() - t
    gen_s = g.gen_s

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize()

    def step(H, out_bufs=None):
        """One pass of the hot path: every algorithm to convergence."""
        res = {}
        for a in algos:
            H.run(a, 0)
            st = H.stats()
            res[a] = st
            if out_bufs is not None:
                H.values_into(out_bufs[a])
        return res

    # ---- warm-up ----
    out_bufs = {a: np.empty(g.V, dtype=np.float32 if a == "pr" else np.uint32) for a in algos}
    for _ in range(args.warmup):
        step(G)
    # edges per step (GTEPS_in): reached out-degrees for SSSP/BFS, E for PR/CC
    edges_per = {}
    for a in algos:
        G.run(a, 0)
        if a in ("sssp", "bfs"):
            edges_per[a] = reached_edges(g, G.values())
        else:
            edges_per[a] = g.E

    st0 = G.stats()
    calib = {"link_gbs": st0["cal_link_gbs"], "thpt_cpt_gbs": st0["cal_cpt_gbs"],
             "zc_request_ns": st0["cal_zc_req_ns"], "zc_line_ns": st0["cal_zc_line_ns"]}
    # ---- timed region ----
    cur = torch.cuda.current_stream()
    times, per_algo_ms, launches = [], {a: [] for a in algos}, 0
    eng_ms = np.zeros(8)
    eng_launch = np.zeros(8, dtype=np.int64)
    eng_chunks = np.zeros(8, dtype=np.int64)
    eng_edges = np.zeros(8, dtype=np.int64)
    link_bytes = 0
    iters = {a: 0 for a in algos}
    exch = {a: None for a in algos}
    detail = {}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            barrier()
            t_ev = []
            for a in algos:
                s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_ev.record(cur)
                G.run(a, 0)                     # blocking: returns after its streams finished
                e_ev.record(cur)
                t_ev.append((a, s_ev, e_ev))
                st = G.stats()
                launches += st["kernel_launches"]
                eng_ms += np.array(st["eng_ms"])
                eng_launch += np.array(st["eng_launches"])
                eng_chunks += np.array(st["eng_chunks"])
                eng_edges += np.array(st["eng_edges"])
                link_bytes += st["bytes_filter"] + st["bytes_compaction"] + st["bytes_zerocopy"]
                iters[a] = st["iterations"]
                exch[a] = {"sparse_iters": st["exch_sparse"], "dense_iters": st["exch_dense"],
                           "bytes_per_rank": st["exch_bytes"]}
                if args.detail_out:
                    detail[a] = {"stats": st, "iter_log": G.iter_log()}
            barrier()
            tot = 0.0
            for a, s_ev, e_ev in t_ev:
                ms = s_ev.elapsed_time(e_ev)
                per_algo_ms[a].append(ms)
                tot += ms
            times.append(tot)
    step_ms = float(np.mean(times))
    if multi:
        tt = torch.tensor([step_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
    edges_step = sum(edges_per.values())
    value = edges_step / (step_ms / 1e3) / 1e9

    # ---- e2e: the public API with host buffers (load from host + run + results to host) ----
    e2e = None
    if args.e2e_steps > 0:
        G.close()
        # the contract's inputs live in pinned host memory: page-lock the caller's CSR
        # arrays once, outside the timed region (hyt_load_csr then reads them in place)
        pinned = pin_host(g.host_arrays())
        e2e_ms, e2e_load_s = [], []
        for _ in range(args.e2e_steps):
            barrier()
            s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_ev.record(cur)
            H = new_handle()
            tl = time.perf_counter()
            g.load(H)
            e2e_load_s.append(time.perf_counter() - tl)
            step(H, out_bufs)
            e_ev.record(cur)
            barrier()
            e2e_ms.append(s_ev.elapsed_time(e_ev))
            H.close()
        em = float(np.mean(e2e_ms))
        if multi:
            tt = torch.tensor([em], device=f"cuda:{local}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            em = float(tt.item())
        h2d = sum(a.nbytes for a in g.host_arrays() if a is not None)
        unpin_host(pinned)
        e2e = {"value": edges_step / (em / 1e3) / 1e9, "unit": "GTEPS", "ms_per_step": em,
               "steps": len(e2e_ms), "step_ms": [float(x) for x in e2e_ms],
               "load_s": float(np.mean(e2e_load_s)),
               "inputs_pinned": len(pinned) == len([a for a in g.host_arrays() if a is not None]),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(4 * g.V * len(algos)),
               "includes": ("hyt_load_shard_begin + hyt_load_shard_rows from this rank's pinned rows" if g.shard else
                            "hyt_load_csr from pinned host arrays") +
                           " (GPU hub sort + relabel into the library's pinned edge store) + runs + hyt_get_values",
               "note": "the caller's arrays are page-locked once outside the timed region (inputs in pinned host memory)"}
    else:
        G.close()

    if rank != 0:
        if multi:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ----
    pk = peaks()
    hbm_peak = float(pk.get("hbm_gbs", 6650.0))
    h2d_peak = measured_h2d_gbs(local)
    tags = hyt.TAGS
    kernel_tags = [1, 2, 3, 4, 5]          # relax: filter, compaction, zero-copy, resident, recompute

    traffic_ratio, traffic_src = {}, None
    tr_files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                             "r*_relax_traffic.json")))
    if tr_files:
        try:
            traffic_ratio = json.load(open(tr_files[-1]))["ratio"]
            traffic_src = "profiles/" + os.path.basename(tr_files[-1])
        except (OSError, ValueError, KeyError):
            traffic_ratio = {}

    pattern, pattern_src = None, None
    pf = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_scatter_bench.json")))
    if pf:
        try:
            pattern = json.load(open(pf[-1]))
            pattern_src = "profiles/" + os.path.basename(pf[-1])
            if "uniform_l2_resident" not in pattern:
                pattern = None
        except (OSError, ValueError):
            pattern = None

    # the L2 reduction ceiling swept over launch shapes and PTX forms (tools/red_ceiling.cu):
    # the best rate any configuration reached into an L2-resident array
    red_ceiling, red_src = None, None
    rf = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_red_ceiling.json")))
    if rf:
        try:
            red_ceiling = max(r["g_per_s"] for r in json.load(open(rf[-1]))["rows"])
            red_src = "profiles/" + os.path.basename(rf[-1])
        except (OSError, ValueError, KeyError):
            red_ceiling = None

    def tag_roof(i):
        if eng_launch[i] == 0:
            return None
        avg_s = eng_ms[i] / 1e3 / eng_launch[i]
        if i == 3:   # zero-copy relax: host-link bound; algorithmic bytes = 16-B chunks read over PCIe
            alg = eng_chunks[i] * 16 / eng_launch[i]
            r = {"kernel": "k_relax<zerocopy>", "bound": "pcie", "peak": h2d_peak,
                 "peak_source": "pinned H2D copy bandwidth measured in this run"}
        else:        # HBM-side relax: edge chunks + 4-B destination access per edge
            alg = (eng_chunks[i] * 16 + eng_edges[i] * 4) / eng_launch[i]
            r = {"kernel": f"k_relax<{tags[i]}>", "bound": "hbm", "peak": hbm_peak,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("fallback") else "")}
        r.update({"achieved": alg / avg_s / 1e9, "unit": "GB/s", "bytes_per_launch": alg,
                  "avg_launch_ms": avg_s * 1e3, "launches": int(eng_launch[i]),
                  "share_of_kernel_time": float(eng_ms[i] / max(1e-9, eng_ms[kernel_tags].sum()))})
        r["frac"] = r["achieved"] / r["peak"]
        if i != 3 and pattern:
            # the same launches against the access pattern's own ceiling on this GPU:
            # one random 4-B destination access per edge into an L2-resident array
            # (tools/scatter_bench.cu; red.add.f32 for PR, a load for the min-algorithms)
            ceil_red = pattern["uniform_l2_resident"]["red_add"]["gedges_s"]
            if red_ceiling:
                ceil_red = max(ceil_red, red_ceiling)
            ceil_ld = pattern["uniform_l2_resident"]["ld"]["gedges_s"]
            eps = eng_edges[i] / eng_launch[i] / avg_s / 1e9
            r["access_pattern"] = {"achieved_gedges_s": eps, "ceiling_red_add_gedges_s": ceil_red,  # hub-block edges included
                                   "frac_of_red_add_ceiling": eps / ceil_red,
                                   "ceiling_load_gedges_s": ceil_ld,
                                   "source": pattern_src + (f" + {red_src}" if red_src else ""),
                                   "note": "random 4-B destination accesses per second; the HBM-copy frac above "
                                           "counts them as 4 B each"}
        r["traffic"] = None
        kind = {1: "filter", 5: "filter", 4: "resident"}.get(i)
        if kind and kind in traffic_ratio:
            # DRAM bytes per algorithmic byte of this launch kind, from the committed
            # ncu capture (tools/traffic_run.py), scaled to this run's average launch
            r["traffic"] = traffic_ratio[kind] * alg
            r["traffic_source"] = f"{traffic_src} (dram/alg = {traffic_ratio[kind]:.3f}, {kind} launches)"
        return r

    dom = max(kernel_tags, key=lambda i: eng_ms[i])
    roof = tag_roof(dom)
    kernels = {tags[i]: tag_roof(i) for i in kernel_tags if eng_launch[i]}
    total_s = sum(times) / 1e3
    host_link = {"bytes": int(link_bytes), "achieved": link_bytes / total_s / 1e9, "peak": h2d_peak,
                 "unit": "GB/s", "frac": link_bytes / total_s / 1e9 / h2d_peak,
                 "note": "algorithmic host-link bytes (filter spans + compacted chunks + zero-copy lines) / step time"}

    extras = None
    if not multi and not args.no_extras and args.shift == 0 and args.config == "tw":
        extras = run_extras(hyt, local, tw_graph=g.g)

    cpu = None
    if not args.no_cpu_baseline and world == 1:   # the contract: rank 0 at N = 1 only
        if multi:
            args.no_cpu_full = True                   # the sharded workload holds no full CSR
        try:
            native = use_native_oracle()
            cpu = cpu_oracle_sample(args.config, max(args.shift, args.cpu_shift), algos)
            cpu.update({"host": host_cpu(), "build": f"gcc -O3 -march=native ({os.path.basename(native)})"})
            if not args.no_cpu_full:
                cpu["full_size"] = cpu_oracle_full_sssp(g.g)
        except Exception as ex:
            cpu = {"error": repr(ex)}

    per_algo = {}
    for a in algos:
        ms = float(np.mean(per_algo_ms[a]))
        per_algo[a] = {"time_to_converge_s": ms / 1e3, "median_s": float(np.median(per_algo_ms[a])) / 1e3,
                       "runs_s": [x / 1e3 for x in per_algo_ms[a]],
                       "gteps": edges_per[a] / (ms / 1e3) / 1e9,
                       "edges": int(edges_per[a]), "iterations": int(iters[a])}
        if multi:
            per_algo[a]["exchange"] = exch[a]
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32(sssp)+f32(pr)", "data": "synthetic",
        "config": {"workload": workload_desc(args.config, args.shift, algos),
                   "budget_gb": args.budget_gb, "engine_mode": args.engine, "partition_bytes": 32 << 20,
                   "params": args.set,
                   "cost_model": "cost_model=1: calibrated on this box for SSSP/BFS/CC, the paper's PCIe-3 rule for PR (SURVEY §8f #2)",
                   "calibration": calib,
                   "parallelism": (f"vertex-range x{world}" + (" (NCCL)" if multi else "")) if multi else "single GPU",
                   "l2": L2_NOTE, "degree_stats": dstats},
        "per_algo": per_algo,
        "roofline": roof,
        "kernels": kernels,
        "host_link": host_link,
        "engine_ms": {tags[i]: float(eng_ms[i]) for i in range(8)},
        "cpu_baseline": cpu,
        "extras": extras,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "setup_s": {"generate": gen_s, "load": load_s},
    }
    s = json.dumps(line)
    print(s, flush=True)
    if args.detail_out:
        with open(args.detail_out, "w") as f:
            json.dump({"line": line, "detail": detail}, f)
    if args.json_out:
        with open(args.json_out, "w") as f:
            f.write(s + "\n")
    if multi:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
