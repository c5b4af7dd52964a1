"""Times attncache_search alone on BASELINE.json configs[4] (1M x 1024 bf16 features) at one batch size and
prints QPS and the HBM / tensor roofline fractions.  Usage: python scripts/search_bench.py [B] [iters]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = synth.CONFIGS["search_sweep"]
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, "cuda")
db = ac.Database(ctx, x)
q, pos, _ = synth.queries(cfg, "cuda", B=B)
idx, score, hit = ac.attncache_search(db, q, cfg.tau)
for _ in range(2):
    ac.attncache_search(db, q, cfg.tau, idx, score, hit)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ac.attncache_search(db, q, cfg.tau, idx, score, hit)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
flops, nbytes = 2.0 * B * cfg.N * cfg.D, (cfg.N + B) * cfg.D * 2 + 8 * B
print(f"search B={B} N={cfg.N} D={cfg.D}: {ms:.3f} ms  {B / ms * 1e3:.0f} qps  {flops / ms / 1e9:.1f} TFLOP/s "
      f"(tensor frac {flops / ms / 1e9 / pk['bf16_tflops']:.3f})  hbm frac {nbytes / ms / 1e6 / pk['hbm_gbs']:.3f}  "
      f"hits {int(hit.sum())}/{len(pos)}")
