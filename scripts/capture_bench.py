"""Times attncache_capture_maps alone (PACKED bf16 maps of `rows` prefills of a config) and prints the
HBM roofline fraction on Q + K read and the packed maps written."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):  # an out-of-tree experiment build
    ac.lib_path = os.environ["ATTNCACHE_LIB"]

name = sys.argv[1] if len(sys.argv) > 1 else "llama32_1b"
cfg = synth.CONFIGS[name]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B - cfg.n_hit
ctx = ac.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
Q, K = (torch.randn(rows, cfg.L, cfg.H, cfg.S, cfg.d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
P = ac.attncache_packed_map_elems(cfg.S)
out = torch.empty(rows, cfg.L, cfg.H, P, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    ac.attncache_capture_maps(ctx, Q, K, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ac.attncache_capture_maps(ctx, Q, K, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nbytes = rows * cfg.L * cfg.H * (2 * cfg.S * cfg.d * 2 + P * 2)
print(f"capture {name} rows={rows}: {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s")
