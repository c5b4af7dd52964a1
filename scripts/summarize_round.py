#!/usr/bin/env python
"""Writes profiles/<tag>_summary.md (+ trimmed raw CSVs) from scripts/profile_round.sh's gpurun_out/ files and
updates profiles/traffic.json (per-launch DRAM bytes used by bench.py's roofline.traffic).

    python scripts/summarize_round.py r01c
"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import summarize_ncu as S  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
KEEP = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput',
        'sm__pipe_tensor_cycles_active', 'sm__inst_executed_pipe_xu', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'lts__t_sector_hit_rate', 'smsp__issue_active', 'sm__throughput', 'launch__shared_mem']
reps = [("configs[1] bench", "full_c1"), ("configs[3] misses", "attend_long_prefill"),
        ("configs[2] misses", "attend_llama3_8b"), ("configs[1] capture", "capture_c1")]
lines = [f"# {tag} ncu summary", "", "Commands: `scripts/profile_round.sh " + tag + "` (each profiled command first ran "
         "plain and exited 0).", "", "## Launch list, configs[1] (`python bench.py --steps 3 --warmup 3 "
         "--no-cpu-baseline --no-search-sweep`, library kernels only; cold-cache, serialised)", "",
         "| kernel | launches | mean us | min us | max us |", "|---|---|---|---|---|"]
lp = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
for k, v in S.launches(lp).items():
    lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {max(v):.2f} |")
subprocess.run(["cp", lp, os.path.join(ROOT, "profiles", f"{tag}_launches.csv")], check=True)
lines += ["", "## Full captures (`ncu --set full --clock-control none --import-source on`)", "",
          "| workload | kernel | duration us | DRAM read GB | DRAM write GB | DRAM % peak | tensor pipe % | regs |",
          "|---|---|---|---|---|---|---|---|"]
tp = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(tp))
for label, name in reps:
    rep = os.path.join(ROOT, "gpurun_out", f"{tag}_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    keep = [i for i, h in enumerate(rows[0]) if any(h.startswith(k) for k in KEEP)]
    out = os.path.join(ROOT, "profiles", f"{tag}_{name}_raw.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        for r in rows:
            w.writerow([r[i] for i in keep])
    seen = set()
    for d in S.full(out):
        k = S.short(d["Kernel Name"][0])
        if k in seen:
            continue
        seen.add(k)
        rd, wr = S.val(d, "dram__bytes_read.sum"), S.val(d, "dram__bytes_write.sum")
        lines.append(f"| {label} | {k} | {S.val(d, 'gpu__time_duration.sum') * 1e6:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                     f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]):.1f} | "
                     f"{float(d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'][0]):.1f} | "
                     f"{d['launch__registers_per_thread'][0]} |")
        if name == "full_c1":
            kind = "apply" if "apply" in k else "attend" if "attend" in k else "search" if "search" in k else None
            if kind:
                traffic["llama32_1b"][kind] = rd + wr
json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
