"""Times attncache_apply_cached alone at a config's shape (PACKED bf16 DB of N entries, `hits` rows each
hitting a distinct entry) and prints the HBM roofline fraction on the algorithmic bytes (triangle of the
maps + V + O).  Usage: python scripts/apply_bench.py [config] [hits] [N] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):  # an out-of-tree experiment build
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
cfg = synth.CONFIGS[name]
hits = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_hit
N = int(sys.argv[3]) if len(sys.argv) > 3 else max(hits, 8)
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
ctx = ac.Context(0)
dev = "cuda"
x = synth.features(cfg.with_(N=N), 0, N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), N, cfg.L, cfg.H, cfg.S, torch.bfloat16, dev,
                       chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
idx = torch.randperm(N, generator=torch.Generator().manual_seed(0))[:hits].to(dev)
g = torch.Generator(device=dev).manual_seed(1)
V = torch.randn(hits, cfg.L, cfg.H, cfg.S, cfg.d, device=dev, generator=g).to(torch.bfloat16)
O = torch.empty_like(V)
for _ in range(3):
    ac.attncache_apply_cached(db, idx, V, O)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ac.attncache_apply_cached(db, idx, V, O)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
tri = cfg.S * (cfg.S + 1) // 2
nbytes = hits * cfg.L * cfg.H * (tri * 2 + 2 * cfg.S * cfg.d * 2)
print(f"apply {name} hits={hits} N={N}: {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s")
