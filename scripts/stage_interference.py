"""Does the A.V kernel slow the miss attention that follows it in the step?  Times attend_full (configs[1]
misses) alone in a loop and right after an apply_cached call, with CUDA events around attend_full only.
    python scripts/stage_interference.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama32_1b"]
dev = torch.device("cuda", 0)
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                       synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
O = torch.empty_like(V)
idx, score, hit = PrefillStep(ctx, db, cfg.tau).search(q)
n = 30
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for mode in ("attend alone", "attend after apply", "apply alone", "apply after attend"):
    for k in range(n + 3):
        if mode == "attend after apply":
            ac.attncache_apply_cached(db, idx, V, O, hit=hit)
        if mode == "apply after attend":
            ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
        e = ev[k - 3] if k >= 3 else None
        if e:
            e[0].record()
        if mode.startswith("attend"):
            ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
        else:
            ac.attncache_apply_cached(db, idx, V, O, hit=hit)
        if e:
            e[1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    print(f"{cfg.name} {mode}: median {ts[n // 2]:.4f} ms  min {ts[0]:.4f}")
