#!/usr/bin/env python
"""One-line summary of a bench.py JSON line (stdin)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
sp = d.get("speedup_vs_full_attention", {})
st = d.get("stages", {})
print("tok/s %.4g ms %.4f | search %.4f apply %.4f (frac %.3f) attend %.4f (hbm %.3f) | full %.4f x%.3f eager %s x%s | e2e %s"
      % (d["value"], d["ms_per_step"], st.get("search", {}).get("ms", 0), d["roofline"]["avg_launch_ms"],
         d["roofline"]["frac"], st.get("attend_full_misses", {}).get("ms", 0),
         st.get("attend_full_misses", {}).get("hbm_frac", 0), sp.get("full_attention_ms", 0), sp.get("batch", 0),
         sp.get("eager_torch_attention_ms"), sp.get("batch_vs_eager_torch"), d.get("e2e", {}).get("value")))
if "capture_misses" in st:
    c = st["capture_misses"]
    print("  capture (f1) %.4f ms hbm %.3f %s" % (c["ms"], c["hbm_frac"], c["variant"]))
if "eq5_block" in d:
    e = d["eq5_block"]
    print("  eq5 block (one layer): full %.4f ms cached %.4f ms (x%.2f)  all-hit %.4f ms (x%.2f)" % (
        e["layer_full_ms"], e["layer_cached_ms"], e["speedup_batch"], e["layer_all_hits_ms"], e["speedup_per_hit"]))
for p in d.get("search_sweep", {}).get("points", []):
    print("  search B=%5d  %.4f ms  qps %.4g  hbm %.3f tensor %.3f hits %d/%d" % (
        p["B"], p["ms"], p["qps"], p["hbm_frac"], p["tensor_frac"], p["hits"], p["planted_hits"]))
if "cpu_baseline" in d:
    print("  cpu_baseline", d["cpu_baseline"])
print("  clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
