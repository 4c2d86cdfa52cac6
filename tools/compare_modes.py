#!/usr/bin/env python
"""Hybrid vs the pure engines of the same build (BASELINE.json target: the hybrid
beats pure-explicit and pure-zero-copy on every oversubscribed config), and the
resident build extension.

  python tools/compare_modes.py --config tw --budgets 16,4 --algos sssp,pr \
         --modes hybrid,filter,compaction,zerocopy --out gpurun_out/modes.json

For every (budget, algorithm, mode): warm-up run, then `--runs` timed runs of
hyt_run (CUDA events around the blocking call); reports time-to-converge, GTEPS,
iterations, host-link bytes / edge volume (the Table VI analog) and per-engine
kernel times.
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
    ap.add_argument("--budgets", default="16,4")
    ap.add_argument("--algos", default="sssp,pr")
    ap.add_argument("--modes", default="hybrid,filter,compaction,zerocopy,hybrid+cache")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/modes.json")
    a = ap.parse_args()
    import torch
    import hytgen
    import paper_2208_14935_b200 as hyt
    t = time.time()
    g = hytgen.make(a.config, shift=a.shift, weighted=True)
    gen_s = time.time() - t
    deg = np.diff(g.off.astype(np.int64))
    results = {"config": a.config, "shift": a.shift, "V": g.V, "E": g.E, "generate_s": gen_s, "rows": []}
    for b in [float(x) for x in a.budgets.split(",")]:
        G = hyt.Graph(device=0, budget=int(b * (1 << 30)))
        G.load(g.off, g.nbr, g.w, symmetric=bool(getattr(g, "symmetric", False)))
        for algo in a.algos.split(","):
            d1 = 8 if algo == "sssp" else 4
            edge_vol = g.E * d1
            for mode in a.modes.split(","):
                row = {"budget_gb": b, "algo": algo, "mode": mode}
                try:
                    G.set("edge_cache", 1 if "+cache" in mode else 0)
                    G.set("cpu_cost", 1 if "+cpu" in mode else 0)
                    G.set("cost_model", 2 if "+cal" in mode else 0)
                    zw = [x for x in mode.split("+") if x.startswith("zw")]
                    G.set("zc_weight", float(zw[0][2:]) if zw else 1.0)
                    G.set("direction", 2 if "+pullall" in mode else 1 if "+pull" in mode else 0)
                    G.set("engine_mode", mode.split("+")[0])
                    for tok in mode.split("+")[1:]:
                        if "=" in tok:                 # "+key=value": any library parameter
                            k, v = tok.split("=")
                            G.set(k, float(v))
                    G.run(algo, 0)                 # warm-up (builds the run context)
                    vals = G.values()
                    edges = int(deg[vals != 0xFFFFFFFF].sum()) if algo in ("sssp", "bfs") else g.E
                    ms = []
                    for _ in range(a.runs):
                        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        torch.cuda.synchronize()
                        s.record()
                        G.run(algo, 0)
                        e.record()
                        torch.cuda.synchronize()
                        ms.append(s.elapsed_time(e))
                    st = G.stats()
                    link = st["bytes_filter"] + st["bytes_compaction"] + st["bytes_zerocopy"]
                    row.update({"ms": float(np.mean(ms)), "gteps": edges / (np.mean(ms) / 1e3) / 1e9,
                                "iterations": st["iterations"], "transfer_over_edge_volume": link / edge_vol,
                                "link_gbs": link / (np.mean(ms) / 1e3) / 1e9,
                                "parts_f": st["parts_filter"], "parts_c": st["parts_compaction"],
                                "parts_z": st["parts_zerocopy"], "parts_r": st["parts_resident"],
                                "pull_iters": st["pull_iters"], "um_balloon_bytes": st["um_balloon_bytes"],
                                "eng_ms": dict(zip(hyt.TAGS, st["eng_ms"])),
                                "device_bytes_peak": st["device_bytes_peak"],
                                "calibration": [st["cal_link_gbs"], st["cal_cpt_gbs"], st["cal_zc_req_ns"],
                                                st["cal_zc_line_ns"]]})
                except hyt.HytError as ex:
                    row["error"] = str(ex)
                print(json.dumps(row), flush=True)
                results["rows"].append(row)
        G.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
