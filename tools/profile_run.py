#!/usr/bin/env python
"""Short, self-contained run of the hot path for ncu captures (one GPU).

  python tools/profile_run.py --config tw --shift 2 --algo pr --engine hybrid --runs 2

Generates the workload (seeded, same recipe as bench.py), loads it once and runs
the algorithm `runs` times.  Prints per-engine kernel times from the library's
CUDA-event counters so a profile can be related to the bench's numbers.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tw")
    ap.add_argument("--shift", type=int, default=2)
    ap.add_argument("--algo", default="pr")
    ap.add_argument("--engine", default="hybrid")
    ap.add_argument("--budget-gb", type=float, default=16.0)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--part", type=int, default=32 << 20)
    ap.add_argument("--set", action="append", default=[], help="key=value library parameter")
    a = ap.parse_args()
    import hytgen
    import paper_2208_14935_b200 as hyt
    t = time.time()
    g = hytgen.make(a.config, shift=a.shift, weighted=True)
    print(f"generated {g.V} V {g.E} E in {time.time() - t:.1f}s", flush=True)
    G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)))
    G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
    G.set("engine_mode", a.engine)
    G.set("partition_bytes", a.part)
    for kv in a.set:
        k, v = kv.split("=")
        G.set(k, float(v))
    for r in range(a.runs):
        G.run(a.algo, 0)
        st = G.stats()
        print(json.dumps({"run": r, "ms": st["time_ns"] / 1e6, "iterations": st["iterations"],
                          "eng_ms": dict(zip(hyt.TAGS, st["eng_ms"])),
                          "eng_launches": dict(zip(hyt.TAGS, st["eng_launches"])),
                          "bytes_f": st["bytes_filter"], "bytes_c": st["bytes_compaction"],
                          "bytes_z": st["bytes_zerocopy"], "launches": st["kernel_launches"]}), flush=True)
    G.close()


if __name__ == "__main__":
    main()
