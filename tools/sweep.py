#!/usr/bin/env python
"""A/B sweep of library parameters on one loaded graph (one GPU, CUDA-event timing).

  python tools/sweep.py --config tw --algos sssp,pr --engines resident,hybrid \
      --variants "relax_hot=0;relax_hot=1" --runs 2 --out gpurun_out/sweep.json

Each variant is a comma-separated list of key=value library parameters applied on
top of the defaults.  Per (engine, algo, variant): one warm-up run, then `runs`
timed runs; prints the min time, iterations and per-engine kernel milliseconds.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


DEFAULTS = {"relax_hot": 1, "relax_ctas_per_sm": 2, "zc_ctas_per_sm": 1, "edge_cache": 0, "relax_bands": 1,
            "relax_threads": 0, "relax_hot_v": 16384,
            "cost_model": 1, "recompute": 1, "priority": -1, "streams": 4, "k": 4, "exchange": 1,
            "partition_bytes": 32 << 20, "epsilon": 1e-5, "zc_ctas": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tw")
    ap.add_argument("--shift", type=int, default=0)
    ap.add_argument("--algos", default="sssp,pr")
    ap.add_argument("--engines", default="resident,hybrid")
    ap.add_argument("--variants", default="relax_hot=0;relax_hot=1")
    ap.add_argument("--budget-gb", type=float, default=16.0)
    ap.add_argument("--resident-budget-gb", type=float, default=100.0)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import hytgen
    import paper_2208_14935_b200 as hyt
    algos = a.algos.split(",")
    t = time.time()
    g = hytgen.make(a.config, shift=a.shift, weighted=("sssp" in algos))
    res = {"config": a.config, "shift": a.shift, "V": g.V, "E": g.E, "generate_s": time.time() - t, "rows": []}
    for engine in a.engines.split(","):
        budget = a.resident_budget_gb if engine == "resident" else a.budget_gb
        G = hyt.Graph(device=0, budget=int(budget * (1 << 30)))
        G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
        for variant in a.variants.split(";"):
            G.set("engine_mode", engine)
            kvs = [kv.split("=") for kv in variant.split(",") if kv]
            for k, v in kvs:
                G.set(k, float(v))
            for algo in algos:
                G.run(algo, 0)
                best = None
                for _ in range(a.runs):
                    torch.cuda.synchronize()
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    G.run(algo, 0)
                    e.record()
                    torch.cuda.synchronize()
                    ms = s.elapsed_time(e)
                    st = G.stats()
                    row = {"engine": engine, "variant": variant, "algo": algo, "ms": ms,
                           "iterations": st["iterations"],
                           "eng_ms": {k: round(v, 3) for k, v in zip(hyt.TAGS, st["eng_ms"]) if v},
                           "eng_launches": {k: v for k, v in zip(hyt.TAGS, st["eng_launches"]) if v}}
                    if best is None or ms < best["ms"]:
                        best = row
                print(json.dumps(best), flush=True)
                res["rows"].append(best)
            for k, _ in kvs:       # back to the default for the next variant (tuning keys only)
                G.set(k, DEFAULTS[k])
        G.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
