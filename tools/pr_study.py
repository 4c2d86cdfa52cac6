#!/usr/bin/env python
"""Delta-PageRank convergence study on the TW workload (bench configuration:
16 GB budget, hybrid): iteration count, time and host-link transfer over repeated
runs, per cost model and epsilon, plus one per-iteration log per setting.

  python tools/pr_study.py --reps 10 --out gpurun_out/pr_study.json
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
    ap.add_argument("--shift", type=int, default=0)
    ap.add_argument("--budget-gb", type=float, default=16)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--settings", default="cost_model=1;cost_model=0;cost_model=1,epsilon=1e-5;cost_model=0,epsilon=1e-5")
    ap.add_argument("--out", default="gpurun_out/pr_study.json")
    a = ap.parse_args()
    import hytgen
    import oracle
    import paper_2208_14935_b200 as hyt
    g = hytgen.make(a.config, a.shift)
    want = None
    if a.shift >= 2:
        want, _ = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-10)
    G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)))
    G.load(g.off, g.nbr)
    out = {"config": a.config, "shift": a.shift, "budget_gb": a.budget_gb, "E": g.E, "rows": {}}
    for setting in a.settings.split(";"):
        kv = dict(x.split("=") for x in setting.split(","))
        for k, v in kv.items():
            G.set(k, float(v))
        G.run("pr")                        # warm (context + calibration)
        rows = []
        for r in range(a.reps):
            t = time.perf_counter()
            G.run("pr")
            ms = (time.perf_counter() - t) * 1e3
            st = G.stats()
            row = {"ms": ms, "iterations": st["iterations"],
                   "xfer_over_edges": (st["bytes_filter"] + st["bytes_compaction"] + st["bytes_zerocopy"]) / (4 * g.E),
                   "parts_fcz": [st["parts_filter"], st["parts_compaction"], st["parts_zerocopy"]],
                   "edges_relaxed": st["edges_relaxed"]}
            if want is not None:
                v = G.values().astype(np.float64)
                row["max_rel_err"] = float(np.max(np.abs(v - want) / want))
            rows.append(row)
            if r == 0:
                out.setdefault("iter_logs", {})[setting] = G.iter_log()
        ms = [x["ms"] for x in rows]
        it = [x["iterations"] for x in rows]
        summ = {"median_ms": float(np.median(ms)), "min_ms": min(ms), "max_ms": max(ms),
                "iters": it, "median_xfer": float(np.median([x["xfer_over_edges"] for x in rows]))}
        if want is not None:
            summ["max_rel_err"] = max(x["max_rel_err"] for x in rows)
        out["rows"][setting] = {"summary": summ, "runs": rows}
        print(setting, json.dumps(summ), flush=True)
        for k in kv:   # back to defaults
            G.set(k, {"cost_model": 1, "epsilon": 1e-5, "zc_weight": 1.0, "relax_bands": 1}.get(k, 0))
    G.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
