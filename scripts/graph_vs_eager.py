"""configs[1] full batch: the step issued eagerly vs replayed as one CUDA graph (pipeline.GraphedPrefillStep)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.pipeline import GraphedPrefillStep, PrefillStep  # noqa: E402

cfg = synth.CONFIGS["llama32_1b"]
dev = torch.device("cuda", 0)
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S, torch.bfloat16, dev, chunk=64)
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
O = torch.empty_like(V)
step = PrefillStep(ctx, db, cfg.tau)
g = GraphedPrefillStep(step, q, Q, K, V)


def timed(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(2):
    print(f"eager {timed(lambda: step(q, Q, K, V, O)):.4f} ms   graph {timed(g.replay):.4f} ms")
