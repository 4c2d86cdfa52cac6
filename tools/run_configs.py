#!/usr/bin/env python
"""Run a BASELINE.json configuration end to end on one GPU and check the results
with the oracle's O(E) certificates (full size) -- for profiles/, not the bench line.

  python tools/run_configs.py --config fr --algos cc,bfs --budget-gb 4 --out gpurun_out/cfg_fr.json
  python tools/run_configs.py --config uk --algos pr,sssp --budget-gb 8 --out gpurun_out/cfg_uk.json
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
    ap.add_argument("--config", default="fr")
    ap.add_argument("--shift", type=int, default=0)
    ap.add_argument("--algos", default="cc,bfs")
    ap.add_argument("--budget-gb", type=float, default=4.0)
    ap.add_argument("--modes", default="hybrid")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--check", type=int, default=1)
    ap.add_argument("--exact", type=int, default=0,
                    help="also compare every vertex with the oracle's own result (minutes at full size)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import hytgen
    import oracle
    import paper_2208_14935_b200 as hyt
    algos = a.algos.split(",")
    t = time.time()
    g = hytgen.make(a.config, shift=a.shift, weighted=("sssp" in algos))
    res = {"config": a.config, "shift": a.shift, "V": g.V, "E": g.E, "generate_s": time.time() - t,
           "budget_gb": a.budget_gb, "degree_stats": g.degree_stats(), "rows": []}
    print(json.dumps({k: v for k, v in res.items() if k != "rows"}), flush=True)
    G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)))
    t = time.time()
    G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
    res["load_s"] = time.time() - t
    deg = np.diff(g.off.astype(np.int64))
    for mode in a.modes.split(","):
        G.set("edge_cache", 1 if "+cache" in mode else 0)
        G.set("cpu_cost", 1 if "+cpu" in mode else 0)
        G.set("cost_model", 2 if "+cal" in mode else 0)
        zw = [x for x in mode.split("+") if x.startswith("zw")]
        G.set("zc_weight", float(zw[0][2:]) if zw else 1.0)
        G.set("direction", 2 if "+pullall" in mode else 1 if "+pull" in mode else 0)
        G.set("engine_mode", mode.split("+")[0])
        for algo in algos:
            G.run(algo, 0)                           # warm-up (run-context build, calibration)
            ms = []
            for _ in range(a.runs):
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                G.run(algo, 0)
                e.record()
                torch.cuda.synchronize()
                ms.append(s.elapsed_time(e))
            vals = G.values()
            st = G.stats()
            edges = int(deg[vals != 0xFFFFFFFF].sum()) if algo in ("bfs", "sssp") else g.E
            d1 = 8 if algo == "sssp" else 4
            link = st["bytes_filter"] + st["bytes_compaction"] + st["bytes_zerocopy"]
            row = {"mode": mode, "algo": algo, "ms": ms, "gteps": edges / (min(ms) / 1e3) / 1e9,
                   "iterations": st["iterations"], "transfer_over_edge_volume": link / (g.E * d1),
                   "parts": [st["parts_filter"], st["parts_compaction"], st["parts_zerocopy"], st["parts_resident"]],
                   "device_bytes_peak": st["device_bytes_peak"],
                   "calibration": [st["cal_link_gbs"], st["cal_cpt_gbs"], st["cal_zc_req_ns"], st["cal_zc_line_ns"]]}
            if a.check:
                t = time.time()
                if algo == "bfs":
                    row["certificate"] = oracle.check_bfs(g.off, g.nbr, 0, vals)
                elif algo == "sssp":
                    row["certificate"] = oracle.check_sssp(g.off, g.nbr, g.w, 0, vals)
                elif algo == "cc":
                    row["certificate"] = oracle.check_cc(g.off, g.nbr, vals)
                else:
                    row["certificate"] = oracle.pr_residual(g.off, g.nbr, vals)
                row["check_s"] = time.time() - t
            if a.exact:
                t = time.time()
                if algo == "bfs":
                    row["equals_oracle"] = bool(np.array_equal(vals, oracle.bfs(g.off, g.nbr, 0)))
                elif algo == "sssp":
                    row["equals_oracle"] = bool(np.array_equal(vals, oracle.sssp(g.off, g.nbr, g.w, 0)))
                elif algo == "cc":
                    row["equals_oracle"] = bool(np.array_equal(vals, oracle.cc(g.off, g.nbr)))
                else:
                    want, _ = oracle.pr_jacobi_pull(g.off, g.nbr, tol=1e-10)
                    row["max_rel_err"] = float(np.max(np.abs(vals.astype(np.float64) - want) / want))
                row["exact_s"] = time.time() - t
            print(json.dumps(row), flush=True)
            res["rows"].append(row)
    G.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
