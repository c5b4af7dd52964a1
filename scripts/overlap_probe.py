"""Step time at a config with apply_cached and attend_full on one stream (sequential, the bench's step) vs
forked onto two streams after the search (the miss attention's CTAs fill SMs as the A.V kernel's retire).

    python scripts/overlap_probe.py [config] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama32_1b"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
dev = torch.device("cuda", 0)
ctx = ac.Context(0)
x = synth.features(cfg, 0, cfg.N, dev)
maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                       synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
q, _, _ = synth.queries(cfg, dev)
Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
O = torch.empty_like(V)
step = PrefillStep(ctx, db, cfg.tau)
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)


def seq():
    idx, score, hit = step.search(q)
    ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)


def fork(attend_first):
    idx, score, hit = step.search(q)
    side.wait_stream(main)
    if attend_first:
        with torch.cuda.stream(side):
            ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
        ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    else:
        ac.attncache_apply_cached(db, idx, V, O, hit=hit)
        with torch.cuda.stream(side):
            ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
    main.wait_stream(side)


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(steps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for name, fn in [("sequential", seq), ("fork apply-first", lambda: fork(False)), ("fork attend-first", lambda: fork(True)),
                 ("sequential", seq)]:
    print(f"{cfg.name} {name}: {timed(fn):.4f} ms/step")
