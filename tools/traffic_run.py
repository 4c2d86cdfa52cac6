#!/usr/bin/env python
"""DRAM traffic of the relax kernel against its algorithmic bytes (bench.py's
`roofline.traffic`).

Step 1 (under ncu, one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k_relax --csv --log-file gpurun_out/traffic_pr.csv \
      python tools/traffic_run.py --algo pr --engine filter --stats-out gpurun_out/traffic_pr.json
Step 2 (here):
  python tools/traffic_run.py --summarize gpurun_out/traffic_pr.csv gpurun_out/traffic_pr.json ... \
      --out profiles/r01_relax_traffic.json

The run is one warm hyt_run on the bench's workload in a pure engine mode, so that
every profiled k_relax launch belongs to the tags counted (filter: the filter and
recompute passes over device-staged edges; resident: the resident pass).  The
ratio DRAM bytes / algorithmic bytes over all launches is what bench.py scales its
per-launch algorithmic bytes by.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TAGS_OF = {"filter": (1, 5), "resident": (4,), "hybrid": (1, 2, 4, 5)}


def run(a):
    import hytgen
    import paper_2208_14935_b200 as hyt
    g = hytgen.make(a.config, shift=a.shift, weighted=True)
    G = hyt.Graph(device=0, budget=int(a.budget_gb * (1 << 30)))
    G.load(g.off, g.nbr, g.w, symmetric=bool(g.symmetric))
    G.set("engine_mode", a.engine)
    # one run (its context build and calibration launch no k_relax)
    tot_chunks = tot_edges = launches = 0
    for _ in range(1):
        G.run(a.algo, 0)
        st = G.stats()
        for t in TAGS_OF[a.engine]:
            tot_chunks += st["eng_chunks"][t]
            tot_edges += st["eng_edges"][t]
            launches += st["eng_launches"][t]
    G.close()
    out = {"config": a.config, "shift": a.shift, "algo": a.algo, "engine": a.engine, "budget_gb": a.budget_gb,
           "relax_launches": launches, "alg_bytes": tot_chunks * 16 + tot_edges * 4,
           "alg_note": "16 B per edge chunk read + 4 B destination access per edge (DESIGN.md §7)"}
    with open(a.stats_out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


def read_csv(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = {}
    for r in rows:
        lid = r["ID"]
        d = per.setdefault(lid, {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                 "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0, "second": 1.0}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    return per


def summarize(pairs, out):
    res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none -k regex:k_relax over tools/traffic_run.py", "runs": []}
    for csv_path, stats_path in pairs:
        st = json.load(open(stats_path))
        per = read_csv(csv_path)
        dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in per.values())
        t = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
        row = dict(st)
        row.update({"ncu_launches": len(per), "dram_bytes": dram, "serialized_s": t,
                    "dram_per_alg_byte": dram / max(1, st["alg_bytes"]),
                    "dram_gbs_serialized": dram / max(1e-12, t) / 1e9})
        res["runs"].append(row)
    by_engine = {}
    for r in res["runs"]:
        e = by_engine.setdefault(r["engine"], {"dram": 0.0, "alg": 0})
        e["dram"] += r["dram_bytes"]
        e["alg"] += r["alg_bytes"]
    res["ratio"] = {k: v["dram"] / max(1, v["alg"]) for k, v in by_engine.items()}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res["ratio"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tw")
    ap.add_argument("--shift", type=int, default=0)
    ap.add_argument("--algo", default="pr")
    ap.add_argument("--engine", default="filter")
    ap.add_argument("--budget-gb", type=float, default=16.0)
    ap.add_argument("--stats-out", default="gpurun_out/traffic.json")
    ap.add_argument("--summarize", nargs="*")
    ap.add_argument("--out", default="profiles/r01_relax_traffic.json")
    a = ap.parse_args()
    if a.summarize:
        it = iter(a.summarize)
        summarize(list(zip(it, it)), a.out)
    else:
        run(a)


if __name__ == "__main__":
    main()
