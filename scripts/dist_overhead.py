"""Breakdown of one owner-affinity step (dist.AffinityPrefill) at world size 1 under torchrun:
GPU time of each phase (CUDA events) and host time of the planning between the search and the local
work.  Usage: torchrun --nproc-per-node 1 --master-addr 127.0.0.1 scripts/dist_overhead.py"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.dist import AffinityPrefill  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("CFG", "llama32_1b")]
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
sizes = [cfg.B]
step = AffinityPrefill(ctx, db, cfg.tau, sizes, bench.apply_bytes_per_hit(cfg), bench.attend_bytes_per_miss(cfg))
for _ in range(3):
    p = step.plan(q)
    step.relocate(X, p)
    step.apply_local(p, p["loc"], V, O, Q, K)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
host = []
res = []
for it in range(10):
    ev[0].record()
    ac.attncache_search_all(db, q, cfg.tau, total=cfg.B)
    ev[1].record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = step.plan(q)  # includes a second search (host planning measured separately below)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ev[2].record()
    step.relocate(X, p)
    ev[3].record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    step.apply_local(p, p["loc"], V, O, Q, K)
    e5.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res.append((ev[0].elapsed_time(ev[1]), (t1 - t0) * 1e3, ev[2].elapsed_time(ev[3]), (t2 - t1) * 1e3,
                e4.elapsed_time(e5), (t3 - t2) * 1e3))
import statistics as st  # noqa: E402
names = ["search_all_gpu_ms", "plan_wall_ms", "relocate_gpu_ms", "relocate_wall_ms", "local_gpu_ms", "local_wall_ms"]
print({n: round(st.median(r[i] for r in res), 4) for i, n in enumerate(names)})
# full steps back to back
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(10):
    p = step.plan(q)
    step.relocate(X, p)
    step.apply_local(p, p["loc"], V, O, Q, K)
s1.record()
torch.cuda.synchronize()
print({"step_ms": s0.elapsed_time(s1) / 10})
dist.destroy_process_group()
