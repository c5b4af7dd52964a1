"""Experiment: A.V (hits, HBM-bound) and miss attention (compute-bound at S = 1024) run concurrently on two
streams with the SMs split between the two persistent kernels (library built with -DSM_EXPERIMENT, CTA
counts from AC_APPLY_SMS / AC_ATTEND_SMS), against the sequential step.
    ATTNCACHE_LIB=ab/smx.so python scripts/sm_split_probe.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402

if os.environ.get("ATTNCACHE_LIB"):
    ac.lib_path = os.environ["ATTNCACHE_LIB"]
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "long_prefill"]
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
idx, score, hit = step.search(q)
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(n):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def seq():
    ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)


def conc():
    side.wait_stream(main)
    ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    with torch.cuda.stream(side):
        ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
    main.wait_stream(side)


os.environ.pop("AC_APPLY_SMS", None)
os.environ.pop("AC_ATTEND_SMS", None)
print(f"{cfg.name} sequential: {timed(seq):.3f} ms  (apply {timed(lambda: ac.attncache_apply_cached(db, idx, V, O, hit=hit)):.3f}, "
      f"attend {timed(lambda: ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)):.3f})")
for k in (16, 24, 32, 40, 48, 64):
    os.environ["AC_APPLY_SMS"], os.environ["AC_ATTEND_SMS"] = str(k), str(148 - k)
    ta = timed(lambda: ac.attncache_apply_cached(db, idx, V, O, hit=hit))
    tt = timed(lambda: ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit))
    print(f"{cfg.name} split apply {k} / attend {148 - k} SMs: concurrent {timed(conc):.3f} ms  (apply alone {ta:.3f}, attend alone {tt:.3f})")
