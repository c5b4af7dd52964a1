#!/usr/bin/env python
"""Summarise ncu output into profiles/: the launch list (per-kernel device times) and the
--set full capture (DRAM traffic, tensor/XU pipe use) of the hot kernels.

    python scripts/summarize_ncu.py <round> <launches.csv> <full_raw.csv> [config]

Writes profiles/r<round>_summary.md and merges per-launch DRAM traffic into profiles/traffic.json
(read by bench.py for roofline.traffic).
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    return re.sub(r"\(.*", "", name).replace("void ", "").split("::")[-1]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        agg.setdefault(short(r[ki]), []).append(float(r[vi].replace(",", "")) / 1e3)
    return agg


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {h: (r[i], units[i]) for i, h in enumerate(hdr)}
        out.append(d)
    return out


def val(d, key, scale=1.0):
    v, u = d[key]
    x = float(v.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u.strip(), 1.0)
    return x * mult * scale


def main():
    rnd, lpath, fpath = sys.argv[1], sys.argv[2], sys.argv[3]
    cfg = sys.argv[4] if len(sys.argv) > 4 else "llama32_1b"
    lines = [f"# Round {rnd} ncu summary ({cfg}, `python bench.py --steps 3 --warmup 3 --no-cpu-baseline`)", ""]
    lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised)",
              "", "| kernel | launches | mean us | min us | max us |", "|---|---|---|---|---|"]
    for k, v in launches(lpath).items():
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.2f} | {min(v):.2f} | {max(v):.2f} |")
    lines += ["", "## Full captures (`ncu --set full --clock-control none`)", "",
              "| kernel | duration us | DRAM read GB | DRAM write GB | DRAM % peak | tensor pipe % | XU % | regs | grid x block |",
              "|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for d in full(fpath):
        name = short(d["Kernel Name"][0])
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        lines.append(
            f"| {name} | {val(d, 'gpu__time_duration.sum') * 1e6:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
            f"{d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]} | "
            f"{d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'][0]} | "
            f"{d['sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'][0]} | "
            f"{d['launch__registers_per_thread'][0]} | {d['launch__grid_size'][0]} x {d['launch__block_size'][0]} |")
        kind = "apply" if "apply" in name else "attend" if "attend" in name else "search" if "search" in name else name
        traffic.setdefault(cfg, {})[kind] = rd + wr
    traffic.setdefault("_note", "per-launch dram__bytes_read.sum + dram__bytes_write.sum from the latest "
                                 "ncu --set full capture (profiles/r*_summary.md)")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    out = os.path.join(ROOT, "profiles", f"r{rnd}_summary.md")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
