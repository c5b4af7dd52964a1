"""Kernel-level breakdown of the Eq. 5 block comparison (block.AttentionBlock) with torch.profiler."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.block import AttentionBlock  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("CFG", "llama32_1b")].with_(L=1)
dev = torch.device("cuda", 0)
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                       synth.torch_dtype(cfg.map_dtype), dev, chunk=64)
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
idx, score, hit = PrefillStep(ctx, db, cfg.tau).search(q)
X, (Wq, Wk, Wv) = synth.block_inputs(cfg, dev)
blk = AttentionBlock(ctx, db, Wq, Wk, Wv, cfg.H, cfg.d, layer=0)
miss_rows = torch.nonzero(hit == 0).flatten()
for _ in range(3):
    blk.full(X)
    blk.cached(X, idx, hit, miss_rows)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
for name, fn in (("full", lambda: blk.full(X)), ("cached", lambda: blk.cached(X, idx, hit, miss_rows))):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
    print("=====", name)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=60))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, "ms", e0.elapsed_time(e1) / 10)
