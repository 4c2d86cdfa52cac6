#!/usr/bin/env python
"""Delta-PageRank f32 error against the oracle's f64 fixed point, binned by in-degree
(f32 atomics accumulate rounding ~ u*sqrt(k) per period at a vertex
with k in-flows; the north star's bar is 1e-4 max relative error per vertex).

  python tools/pr_error.py --config tw --shift 2 --budget-gb 2 --modes hybrid,resident

For each mode: one GPU run (the library default epsilon, 1e-5), then max |r - r*| / r* over all vertices
and per in-degree decade, r* = oracle.pr_jacobi_pull (Jacobi to 1e-11, f64, CPU threads).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tw")
    ap.add_argument("--shift", type=int, default=2)
    ap.add_argument("--budget-gb", type=float, default=2.0)
    ap.add_argument("--modes", default="hybrid,resident")
    ap.add_argument("--out", default="gpurun_out/pr_error.json")
    a = ap.parse_args()
    import hytgen
    import oracle
    import paper_2208_14935_b200 as hyt
    g = hytgen.make(a.config, shift=a.shift)
    t = time.time()
    want, iters = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-11)
    res = {"config": a.config, "shift": a.shift, "V": g.V, "E": g.E, "oracle_s": time.time() - t,
           "oracle_iters": iters, "rows": []}
    indeg = np.bincount(g.nbr, minlength=g.V)
    edges = [0, 1, 10, 100, 1000, 10000, 100000, 1 << 40]
    for mode in a.modes.split(","):
        G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)) if mode != "resident" else 0)
        try:
            G.load(g.off, g.nbr)
            G.set("engine_mode", mode)
            G.run("pr")
            got = G.values().astype(np.float64)
            st = G.stats()
        finally:
            G.close()
        rel = np.abs(got - want) / want
        bins = []
        for lo, hi in zip(edges[:-1], edges[1:]):
            m = (indeg >= lo) & (indeg < hi)
            if m.any():
                bins.append({"indeg": [lo, hi], "vertices": int(m.sum()), "max_rel": float(rel[m].max()),
                             "mean_rel": float(rel[m].mean())})
        row = {"mode": mode, "iterations": st["iterations"], "max_rel": float(rel.max()),
               "argmax_indeg": int(indeg[rel.argmax()]), "bins": bins}
        print(json.dumps(row), flush=True)
        res["rows"].append(row)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
