"""Times attncache_project_features (f2) alone at a config's batch and at B = 8192, as bench.py's project
stage does.  Usage: python scripts/project_bench.py [config] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama32_1b"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ctx = ac.Context(0)
for B in (cfg.B, 1024, 8192):
    h, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=B, device="cuda")
    f = torch.empty(B, cfg.D, dtype=synth.torch_dtype(cfg.feat_dtype), device="cuda")
    for _ in range(3):
        ac.attncache_project_features(ctx, h, W1, b1, W2, b2, out=f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ac.attncache_project_features(ctx, h, W1, b1, W2, b2, out=f)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    E, Hd, D = h.shape[1], W1.shape[0], cfg.D
    print(f"project {cfg.name} B={B} E={E} Hd={Hd} D={D}: {ms * 1e3:.1f} us  "
          f"{2.0 * B * (E * Hd + Hd * D) / (ms * 1e-3) / 1e12:.0f} TFLOP/s")
