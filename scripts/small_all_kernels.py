#!/usr/bin/env python
"""Small end-to-end run of every kernel family and both map layouts (tiny shapes, ragged sizes).
Meant for compute-sanitizer (one tool per invocation), which is closed on the current GPU pool; the
bitwise repeat test and the oracle parity tests stand in for it there."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402

dev = "cuda"
ctx = ac.Context(0)
for name, over in (("tiny", {}), ("llama32_1b", dict(N=8, B=5, L=1, H=4)), ("llama3_8b", dict(N=4, B=3, L=1, H=2)),
                   ("long_prefill", dict(N=2, B=2, L=1, H=1))):
    cfg = synth.CONFIGS[name].with_(**over)
    x = synth.features(cfg, 0, cfg.N, dev)
    dense = synth.maps(cfg, 0, cfg.N, dev)
    for packed in (False, True):
        maps = ac.attncache_pack_maps(dense) if packed else dense
        db = ac.Database(ctx, x, maps, packed=packed, seq_len=cfg.S)
        q, _, _ = synth.queries(cfg, dev)
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
        O = torch.empty_like(V)
        PrefillStep(ctx, db, cfg.tau)(q, Q, K, V, O)
        ac.attncache_apply_cached(db, torch.arange(cfg.B, device=dev) % cfg.N, V, O)
        ac.attncache_fetch_maps(db, cfg.N - 1)
        ctx.sync()
    print(name, "ok", flush=True)
big = synth.CONFIGS["search_sweep"].with_(N=3000)
xb = synth.features(big, 0, big.N, dev)
dbs = ac.Database(ctx, xb)
for B in (1, 100, 300):
    qb, _, _ = synth.queries(big, dev, B=B)
    ac.attncache_search(dbs, qb, big.tau)
ctx.sync()
print("sanitize run complete")
