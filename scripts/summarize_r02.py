#!/usr/bin/env python
"""Summarise round-2 ncu captures (profiles/<P>_*_raw.csv from `ncu -i X.ncu-rep --page raw --csv`) and the
launch list into profiles/<P>_summary.md, and merge per-launch DRAM traffic into profiles/traffic.json.

    python scripts/summarize_r02.py r02a"""
import collections
import csv
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = sys.argv[1] if len(sys.argv) > 1 else "r02a"
M = collections.OrderedDict([
    ("time_us", "gpu__time_duration.sum"),
    ("tensor_pipe_%", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("smem_tc_%", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("xu_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("dram_rd_GB", "dram__bytes_read.sum"),
    ("dram_wr_GB", "dram__bytes_write.sum"),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
])
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "s": 1e6, "Gbyte": 1.0, "Mbyte": 1e-3, "Tbyte": 1e3, "Kbyte": 1e-6, "byte": 1e-9}


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    out = []
    for d in r[2:]:
        rec = {"kernel": re.sub(r"\(.*", "", d[hdr.index("Kernel Name")]).replace("void ", "").replace("(anonymous namespace)::", "")}
        for k, m in M.items():
            cand = [i for i, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if cand:
                i = cand[0]
                v = float(d[i].replace(",", "")) if d[i] else float("nan")
                rec[k] = v * SCALE.get(units[i], 1.0) if k in ("time_us", "dram_rd_GB", "dram_wr_GB") else v
        out.append(rec)
    return out


lines = [f"# ncu summary {P} (one B200; `ncu --set full --clock-control none`; cold-cache, serialised replays)", "",
         "| capture | kernel | " + " | ".join(M) + " |", "|" + "---|" * (len(M) + 2)]
traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{P}_*_raw.csv"))):
    cap = os.path.basename(f)[len(P) + 1:-len("_raw.csv")]
    for rec in rows(f):
        lines.append(f"| {cap} | {rec['kernel']} | " + " | ".join(f"{rec.get(k, float('nan')):.3g}" for k in M) + " |")
        cfg = {"apply_llama3_8b": ("llama3_8b", "apply"), "full_c1": ("llama32_1b", None)}.get(cap)
        if cfg and cfg[1] and "apply_tc" in rec["kernel"]:
            traffic.setdefault(cfg[0], {})[cfg[1]] = (rec["dram_rd_GB"] + rec["dram_wr_GB"]) * 1e9
        if cap == "full_c1" and "apply_tc" in rec["kernel"]:
            traffic.setdefault("llama32_1b", {})["apply"] = (rec["dram_rd_GB"] + rec["dram_wr_GB"]) * 1e9
launch = os.path.join(ROOT, "profiles", f"{P}_launches.csv")
if os.path.exists(launch):
    r = [x for x in csv.reader(open(launch)) if len(x) > 10]
    hdr, data = r[0], r[1:]
    agg = collections.OrderedDict()
    for d in data:
        k = re.sub(r"\(.*", "", d[hdr.index("Kernel Name")])
        agg.setdefault(k, []).append(float(d[hdr.index("Metric Value")].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    lines += ["", f"Launch list ({os.path.basename(launch)}, bench.py at configs[1], all launches of the process):", "",
              "| kernel | launches | mean us | share of kernel time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
json.dump(traffic, open(traffic_path, "w"), indent=1)
open(os.path.join(ROOT, "profiles", f"{P}_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:40]))
