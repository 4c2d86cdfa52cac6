#!/usr/bin/env python
"""Where bench.py's e2e step spends its time: handle creation, hyt_load_csr (with
HYT_VERBOSE phase timers), the first (cold: run-context build) and second (warm)
hyt_run of each algorithm, and hyt_get_values.  Wall clock around each call.

  HYT_VERBOSE=1 python tools/e2e_breakdown.py --config tw
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
    ap.add_argument("--shift", type=int, default=0)
    ap.add_argument("--algos", default="sssp,pr")
    ap.add_argument("--budget-gb", type=float, default=16.0)
    ap.add_argument("--pin", type=int, default=0, help="page-lock the caller arrays first (bench.py's e2e)")
    a = ap.parse_args()
    import numpy as np
    import hytgen
    import paper_2208_14935_b200 as hyt
    g = hytgen.make(a.config, shift=a.shift, weighted=True)
    out = {"pin": a.pin}
    if a.pin:
        from bench import pin_host
        t = time.time()
        out["pinned"] = len(pin_host([g.off, g.nbr, g.w]))
        out["pin_s"] = time.time() - t
    for rep in range(2):
        t = time.time()
        G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)))
        out[f"{rep}:handle_s"] = time.time() - t
        t = time.time()
        G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
        out[f"{rep}:load_s"] = time.time() - t
        for algo in a.algos.split(","):
            for k in ("cold", "warm"):
                t = time.time()
                G.run(algo, 0)
                out[f"{rep}:{algo}_{k}_s"] = time.time() - t
                out[f"{rep}:{algo}_{k}_iters"] = G.stats()["iterations"]
            t = time.time()
            v = np.empty(g.V, dtype=np.float32 if algo == "pr" else np.uint32)
            G.values_into(v)
            out[f"{rep}:{algo}_values_s"] = time.time() - t
        t = time.time()
        G.close()
        out[f"{rep}:close_s"] = time.time() - t
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
