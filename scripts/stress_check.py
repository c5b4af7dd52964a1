"""Runs every tcgen05 kernel family once per repeat on fixed seeded inputs and saves the outputs, for the
schedule-stress comparison of tests/test_gpu_stress.py: the library under ATTNCACHE_LIB (a -DAC_STRESS
build, whose role loops sleep at random) must reproduce the normal build's outputs bit for bit.

    ATTNCACHE_LIB=/path/libattncache.so python scripts/stress_check.py OUT.pt [repeats]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_25979_b200 as ac  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
out_path = sys.argv[1]
repeats = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
ctx = ac.Context(0)


def rnd(shape, seed, dtype=torch.bfloat16, scale=1.0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(shape, device=dev, generator=g) * scale).to(dtype)


def normed(n, D, seed):
    x = rnd((n, D), seed, torch.float32)
    return (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16)


def softmax_maps(n, L, H, S, seed):
    s = rnd((n, L, H, S, S), seed, torch.float32, 2.0)
    s = s.masked_fill(torch.ones(S, S, device=dev, dtype=torch.bool).triu(1), float("-inf"))
    return torch.softmax(s, dim=-1).to(torch.bfloat16)


results = {}
cases = []

# Sizes give every persistent CTA many items (the races a stress build exposes need item switches).
# attention: d = 128 (column-split kernel; S = 1024 and a GQA S = 384 case with a skipped row) and
# d = 64 (two-group kernel)
for name, (rows, L, H, Hkv, S, d) in {"att128": (8, 4, 8, 8, 1024, 128), "att128gqa": (16, 2, 8, 2, 384, 128),
                                      "att64": (16, 4, 8, 8, 256, 64), "att64tail": (8, 2, 8, 8, 200, 64),
                                      "att128tail": (8, 2, 8, 8, 1019, 128)}.items():
    Q = rnd((rows, L, H, S, d), 1)
    K = rnd((rows, L, Hkv, S, d), 2)
    V = rnd((rows, L, Hkv, S, d), 3)
    skip = torch.zeros(rows, dtype=torch.uint8, device=dev)
    skip[1] = 1
    cases.append((name, lambda Q=Q, K=K, V=V, skip=skip: ac.attncache_attend_full(ctx, Q, K, V, torch.zeros_like(Q),
                                                                                 skip=skip)))

# A.V over packed causal maps: d = 64 / S = 128 and d = 128 / S = 256
# (S > 128: the paired-row-block kernel, an odd row-block count and a partial last block included)
for name, (N, B, L, H, S, d) in {"apply64": (16, 64, 4, 8, 128, 64), "apply128": (8, 16, 4, 8, 256, 128),
                                 "apply128pairs": (6, 12, 2, 8, 640, 128), "apply64tail": (6, 12, 2, 8, 584, 64)}.items():
    maps = torch.empty((N, L, H, ac.attncache_packed_map_elems(S)), dtype=torch.bfloat16, device=dev)
    ac.attncache_pack_maps(softmax_maps(N, L, H, S, 4), maps)
    db = ac.Database(ctx, normed(N, 256, 5), maps, packed=True, seq_len=S)
    g = torch.Generator().manual_seed(6)
    idx = torch.randint(0, N, (B,), generator=g).to(dev)
    hit = (torch.rand(B, generator=g) < 0.8).to(torch.uint8).to(dev)
    V = rnd((B, L, H, S, d), 7)
    keep = (db, maps)
    cases.append((name, lambda db=db, idx=idx, hit=hit, V=V, keep=keep: ac.attncache_apply_cached(
        db, idx, V, torch.zeros_like(V), hit=hit)))

# capture (packed maps): d = 64 / S = 128 and d = 128 / S = 1024 (streamed stores)
for name, (rows, L, H, S, d) in {"cap64": (16, 4, 8, 128, 64), "cap128": (4, 2, 8, 1024, 128)}.items():
    Q = rnd((rows, L, H, S, d), 8)
    K = rnd((rows, L, H, S, d), 9)
    cases.append((name, lambda Q=Q, K=K: ac.attncache_capture_maps(ctx, Q, K)))

# search: B = 64 and B = 1024 over 4096 x 1024 bf16 features
x = normed(4096, 1024, 10)
db_s = ac.Database(ctx, x)
for B in (64, 1024):
    q = normed(B, 1024, 11 + B)
    cases.append((f"search{B}", lambda q=q: torch.stack([t.to(torch.float64) for t in ac.attncache_search(db_s, q, 0.5)])))
# the two-query-tile search kernel (B > 128 and enough (pair, entry tile) items): 150,001 entries, B = 300
x2 = normed(150_001, 1024, 12)
db_s2 = ac.Database(ctx, x2)
q2 = normed(300, 1024, 13)
cases.append(("search_pairs", lambda: torch.stack([t.to(torch.float64) for t in ac.attncache_search(db_s2, q2, 0.5)])))

# feature projector (two tcgen05 GEMMs + normalisation)
h = rnd((2048, 2048), 12)
W1, W2 = rnd((1024, 2048), 13, scale=0.03), rnd((1024, 1024), 14, scale=0.03)
b1, b2 = rnd((1024,), 15, torch.float32, 0.1), rnd((1024,), 16, torch.float32, 0.1)
cases.append(("project", lambda: ac.attncache_project_features(ctx, h, W1, b1, W2, b2)))

import time  # noqa: E402
t0 = time.time()
for name, fn in cases:
    outs = []
    for _ in range(repeats):
        outs.append(fn().clone())
        torch.cuda.synchronize()
    ctx.sync()
    results[name] = outs
torch.save({k: [t.cpu() for t in v] for k, v in results.items()}, out_path)
print("ok", len(results), "cases x", repeats, f"{time.time() - t0:.2f} s")
