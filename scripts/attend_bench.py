"""Times attncache_attend_full alone on the miss batch of a config (CUDA events, warm-up, inputs > L2)
and prints achieved TFLOP/s (causal flops 4*d*tri(S) per (row, layer, head)) and HBM GB/s.
Usage: python scripts/attend_bench.py [config] [rows] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):  # an out-of-tree experiment build (ATTNCACHE_BUILD_ROOT / ATTNCACHE_EXTRA_FLAGS)
    ac.lib_path = os.environ["ATTNCACHE_LIB"]

name = sys.argv[1] if len(sys.argv) > 1 else "long_prefill"
cfg = synth.CONFIGS[name]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B - cfg.n_hit
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
ctx = ac.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
shape = (rows, cfg.L, cfg.H, cfg.S, cfg.d)
Q, K, V = (torch.randn(shape, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
O = torch.empty_like(V)
for _ in range(3):
    ac.attncache_attend_full(ctx, Q, K, V, O)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ac.attncache_attend_full(ctx, Q, K, V, O)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
units = rows * cfg.L * cfg.H
flops = units * 4.0 * cfg.d * cfg.S * (cfg.S + 1) / 2
nbytes = units * 4.0 * cfg.S * cfg.d * 2
print(f"{name} rows={rows} S={cfg.S} d={cfg.d}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s  "
      f"{nbytes / ms / 1e6:.1f} GB/s  variant={ac.attncache_variant('attend', V.dtype, cfg.S, cfg.d)}")
