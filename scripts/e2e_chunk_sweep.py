"""e2e (attncache_prefill_host) chunk / depth sweep at one config: the host-buffer step time per (chunk, depth)
against the copy floor (the step's H2D + D2H bytes copied with no kernel).  Usage:
    python scripts/e2e_chunk_sweep.py llama3_8b "4,8,16" "2,4"
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from bench import _copy_bound  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
chunks = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16").split(",")]
depths = [int(c) for c in (sys.argv[3] if len(sys.argv) > 3 else "4").split(",")]
cfg = synth.CONFIGS[name]
dev = "cuda:0"
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                       synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
qh, Qh, Kh, Vh = (t.cpu().pin_memory() for t in (q, Q, K, V))
Oh = torch.empty(V.shape, dtype=V.dtype).pin_memory()
idx, score, hit, _ = ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh)
n_miss = int((hit == 0).sum())
best = None
for c in chunks:
    for dp in depths:
        for _ in range(2):
            ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh, idx=idx, score=score, hit=hit, chunk=c, depth=dp)
        torch.cuda.synchronize()
        n = 5
        t0 = time.perf_counter()
        for _ in range(n):
            ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh, idx=idx, score=score, hit=hit, chunk=c, depth=dp)
        ms = (time.perf_counter() - t0) * 1e3 / n
        print(f"{name} chunk {c:3d} depth {dp}: {ms:8.2f} ms  {cfg.B * cfg.S / ms / 1e3:8.3f} M tok/s", flush=True)
        best = ms if best is None else min(best, ms)
cb = _copy_bound(Vh, V, Qh[:n_miss], Q[:n_miss], Kh[:n_miss], K[:n_miss], Oh, best)
print(f"{name} copy floor {cb['copies_only_ms']:.2f} ms; best step / floor = {cb['copies_only_ms'] / best:.3f}")
