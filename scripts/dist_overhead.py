"""Per-stage cost of the owner-affinity multi-GPU step at world size 1 (the library's collective calls over a
one-rank NCCL communicator) and the ownership balance the placement reaches at g = 2..8 on the config's real
search results; the inputs of DESIGN.md §8's strong-scaling model.
Usage: torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/dist_overhead.py [config]"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.dist import AffinityPrefill, shard_range  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama32_1b"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
ctx = ac.Context.from_process_group(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                       synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
O = torch.empty_like(V)
X = torch.randn(cfg.B, cfg.S, cfg.H * cfg.d, device=dev).to(torch.bfloat16)
hc, mc = bench.apply_bytes_per_hit(cfg), bench.attend_bytes_per_miss(cfg)
step = AffinityPrefill(ctx, db, cfg.tau, [cfg.B], hc, mc)
p = step.plan(q)
for _ in range(3):
    step.relocate(X, p)
    step.apply_local(p, p["loc"], V, O, Q, K)
torch.cuda.synchronize()


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n


out = {"config": cfg.name}
out["search_all_ms"], _ = timed(lambda: ac.attncache_search_all(db, q, cfg.tau, total=cfg.B))
out["local_search_ms"], _ = timed(lambda: ac.attncache_search(ac.Database(ac.Context(0), x), q, cfg.tau), 3)
_, out["plan_wall_ms"] = timed(lambda: step.plan(q))
out["relocate_ms"], _ = timed(lambda: step.relocate(X, p))
out["relocate_bytes"] = X.numel() * X.element_size()
out["local_ms"], _ = timed(lambda: step.apply_local(p, p["loc"], V, O, Q, K))
# ownership balance of the placement on this batch's real decisions at g GPUs (load = algorithmic bytes)
idx, hit = p["idx"].cpu().numpy(), p["hit"].cpu().numpy()
bal = {}
for g in (2, 4, 8):
    sb = [shard_range(cfg.N, g, r)[0] for r in range(g)] + [cfg.N]
    _, load = ac.attncache_affinity_plan(idx, hit, sb, hc, mc)
    bal[g] = float(load.mean() / load.max())
out["placement_balance_mean_over_max"] = bal
print(json.dumps(out))
dist.destroy_process_group()
