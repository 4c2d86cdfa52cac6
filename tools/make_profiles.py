#!/usr/bin/env python
"""Write the round's measurement summary under profiles/ from gpurun_out/ artefacts.

  python tools/make_profiles.py --round 1
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def last_json(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def exec_path(detail_path, out):
    d = json.load(open(detail_path))
    lines = ["# Execution path per iteration (Fig. 7 analog) — TW-shaped graph, 16 GB budget, hybrid\n",
             "Each row: active vertices / edges at the iteration's plan, partitions per engine "
             "(F filter, C compaction, Z zero-copy, R resident), filter units after combination (k = 4), "
             "and host-link bytes per engine.\n"]
    for algo, v in d["detail"].items():
        st = v["stats"]
        lines.append(f"\n## {algo}: {st['iterations']} iterations, {st['time_ns'] / 1e6:.1f} ms, "
                     f"bytes F/C/Z = {st['bytes_filter'] / 1e9:.2f} / {st['bytes_compaction'] / 1e9:.2f} / "
                     f"{st['bytes_zerocopy'] / 1e9:.2f} GB\n")
        lines.append("| it | active V | active E | F | C | Z | R | units | F GB | C GB | Z GB |")
        lines.append("|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
        for r in v["iter_log"]:
            lines.append(f"| {r['iteration']} | {r['active_vertices']} | {r['active_edges']} | {r['parts_f']} | "
                         f"{r['parts_c']} | {r['parts_z']} | {r['parts_r']} | {r['units_f']} | "
                         f"{r['bytes_f'] / 1e9:.2f} | {r['bytes_c'] / 1e9:.2f} | {r['bytes_z'] / 1e9:.2f} |")
    open(out, "w").write("\n".join(lines) + "\n")


def modes(path, out):
    m = json.load(open(path))
    lines = [f"# Hybrid vs pure engines (same build) — {m['config']} ({m['V']} V, {m['E']} E)\n",
             "`tools/compare_modes.py`: one warm-up run then one timed hyt_run per row (CUDA events). "
             "transfer/edge = host-link bytes / (E x d1), the Table VI analog.\n",
             "| budget GB | algo | mode | ms | GTEPS | iterations | transfer/edge | link GB/s | F/C/Z partitions |",
             "|---:|---|---|---:|---:|---:|---:|---:|---|"]
    for r in m["rows"]:
        if "error" in r:
            lines.append(f"| {r['budget_gb']} | {r['algo']} | {r['mode']} | error: {r['error'][:80]} |||||||")
            continue
        lines.append(f"| {r['budget_gb']} | {r['algo']} | {r['mode']} | {r['ms']:.1f} | {r['gteps']:.3f} | "
                     f"{r['iterations']} | {r['transfer_over_edge_volume']:.2f} | {r['link_gbs']:.1f} | "
                     f"{r['parts_f']}/{r['parts_c']}/{r['parts_z']} |")
    open(out, "w").write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    r = f"r{a.round:02d}"
    os.makedirs(P, exist_ok=True)
    for name in ("bench_full.log", "bench_resident.log"):
        src = os.path.join(G, name)
        if os.path.exists(src):
            with open(os.path.join(P, f"{r}_{name.replace('.log', '.json')}"), "w") as f:
                json.dump(last_json(src), f, indent=1)
    if os.path.exists(os.path.join(G, "bench_detail.json")):
        exec_path(os.path.join(G, "bench_detail.json"), os.path.join(P, f"{r}_exec_path_tw.md"))
    for src, dst in (("modes_final.json", "modes_tw"), ("modes.json", "modes_tw")):
        if os.path.exists(os.path.join(G, src)):
            modes(os.path.join(G, src), os.path.join(P, f"{r}_{dst}.md"))
            break
    cfg_lines = ["# Full-size configurations (tools/run_configs.py, warm runs, O(E) certificates where run)\n",
                 "| config | V | E | budget GB | algo | mode | ms (runs) | iterations | transfer/edge | F/C/Z/R partitions | certificate |",
                 "|---|---:|---:|---:|---|---|---|---:|---:|---|---|"]
    for name in ("cfg_fr.json", "cfg_fr_cal.json", "cfg_uk.json", "cfg_uk_cal.json", "cfg_r30s3.json",
                 "cfg_r30s3_cal.json"):
        path = os.path.join(G, name)
        if not os.path.exists(path):
            continue
        d = json.load(open(path))
        for row in d["rows"]:
            cert = row.get("certificate", "")
            if isinstance(cert, dict):
                cert = f"res_l1 {cert['res_l1']:.1f}, max rel res {cert['max_rel_res']:.1e}"
            name_s = d['config'] + (f">>{d['shift']}" if d.get('shift') else "")
            cfg_lines.append(f"| {name_s} | {d['V']} | {d['E']} | {d['budget_gb']} | {row['algo']} | {row['mode']} | "
                             f"{', '.join(f'{x:.1f}' for x in row['ms'])} | {row['iterations']} | "
                             f"{row['transfer_over_edge_volume']:.2f} | {'/'.join(str(x) for x in row['parts'])} | {cert} |")
    open(os.path.join(P, f"{r}_configs_full_size.md"), "w").write("\n".join(cfg_lines) + "\n")
    for src in ("zc_bench.json", "scatter_bench.json", "sweep_hot.json"):
        if os.path.exists(os.path.join(G, src)):
            import shutil
            shutil.copy(os.path.join(G, src), os.path.join(P, f"{r}_{src}"))
    for csvname, tag in (("launches_w1.csv", "launches_bench"),):
        src = os.path.join(G, csvname)
        if os.path.exists(src):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "launches", src],
                                 capture_output=True, text=True).stdout
            open(os.path.join(P, f"{r}_{tag}.md"), "w").write(out)


if __name__ == "__main__":
    main()
