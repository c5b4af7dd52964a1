"""Timeline of the d=128 attention (--split: the default column-split kernel, softmax warp 4 and the MMA thread;
otherwise the two-group kernel, CTA 0, group 0 = warp 4 and group 1 = warp 8, lane 0): builds
the library with -DATT_TRACE out of tree, runs configs[3]'s misses once and prints per-block phase
durations in cycles: wait for S, TMEM load of S, row max, exp + P store, arrive, and the gap to the next."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SPLIT = "--split" in sys.argv
PP = "--pp" in sys.argv
for f in ("--split", "--pp"):
    if f in sys.argv:
        sys.argv.remove(f)
KIND = "s" if SPLIT else ("p" if PP else "")
env = dict(os.environ, ATTNCACHE_BUILD_ROOT="/tmp/atttrace" + KIND,
           ATTNCACHE_EXTRA_FLAGS="-DATT_TRACE " + os.environ.get("TRACE_FLAGS", "") +
           (" -DATT_SPLIT128" if SPLIT else ("" if PP else " -DATT_TWO_GROUP128")))
subprocess.check_call([sys.executable, "-m", "paper_2510_25979_b200.build"], env=env, cwd=ROOT, stdout=subprocess.DEVNULL)
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
ac.lib_path = "/tmp/atttrace" + KIND + "/lib/libattncache.so"
name = sys.argv[1] if len(sys.argv) > 1 else "long_prefill"
cfg = synth.CONFIGS[name]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B - cfg.n_hit
ctx = ac.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
shape = (rows, cfg.L, cfg.H, cfg.S, cfg.d)
Q, K, V = (torch.randn(shape, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
O = ac.attncache_attend_full(ctx, Q, K, V)
torch.cuda.synchronize()
ac.attncache_attend_full(ctx, Q, K, V, O)
torch.cuda.synchronize()
lib = ac.load_library()
if PP:
    sm = np.zeros((256, 8, 5), dtype=np.uint64)
    mm = np.zeros((256, 6), dtype=np.uint64)
    assert lib.attncache_debug_pp_trace(ctypes.c_void_p(sm.ctypes.data), ctypes.c_void_p(mm.ctypes.data)) == 0
    t, m = sm.astype(np.int64), mm.astype(np.int64)
    print("per softmax warp (4-7 group 0 = even blocks, 8-11 group 1 = odd), median cycles over its blocks 20..200:")
    print("  warp: [S wait, load + max, rescale + exp + P store, arrive, gap to next start]")
    for w in range(8):
        bs = np.arange(20 + (w >= 4), 200, 2)
        d = np.diff(t[bs, w], axis=1)
        gap = t[bs[1:], w, 0] - t[bs[:-1], w, 4]
        print(f"  {4 + w}: {np.median(d, axis=0).astype(int).tolist()} gap {int(np.median(gap))}  period/2 blocks "
              f"{int(np.median(np.diff(t[bs, w, 0])))}")
    dm = np.diff(m[20:200, :4], axis=1)
    print("MMA median: P ok -> V ok", int(np.median(m[20:200, 4] - m[20:200, 1])), " V ok -> PV issued",
          int(np.median(m[20:200, 2] - m[20:200, 4])), " PV issued -> K ok", int(np.median(m[20:200, 5] - m[20:200, 2])),
          " K ok -> S issued", int(np.median(m[20:200, 3] - m[20:200, 5])))
    last = np.array([t[b, 4 * (b % 2):4 * (b % 2) + 4, 4].max() for b in range(20, 200)])
    print("MMA median: wait P", int(np.median(dm[:, 0])), " PV issue", int(np.median(dm[:, 1])), " S issue",
          int(np.median(dm[:, 2])), " period", int(np.median(np.diff(m[20:200, 0]))),
          " P-ok after the group's last arrival", int(np.median(m[20:200, 1] - last)))
    base = m[40, 0]
    print("blocks 40..52 rel. MMA wait start of block 40: MMA [wait, P ok, PV, S] | owner warps' [start, S ok, max, P, arr] (warp 4/8)")
    for b in range(40, 52):
        w = 4 * (b % 2)
        print(b, [int(x - base) for x in m[b, :4]], [int(x - base) for x in t[b, w]])
    sys.exit(0)
if SPLIT:
    sm = np.zeros((256, 6), dtype=np.uint64)
    mm = np.zeros((256, 6), dtype=np.uint64)
    assert lib.attncache_debug_split_trace(ctypes.c_void_p(sm.ctypes.data), ctypes.c_void_p(mm.ctypes.data)) == 0
    t, m = sm.astype(np.int64), mm.astype(np.int64)
    d = np.diff(t[:, :5], axis=1)
    per = t[1:, 0] - t[:-1, 0]
    sel = slice(20, 200)
    print(f"softmax warp 4: median cycles wait_S {np.median(d[sel, 0]):.0f}  load+exchange {np.median(d[sel, 1]):.0f}  "
          f"exp+store {np.median(d[sel, 2]):.0f}  arrive {np.median(d[sel, 3]):.0f}  period {np.median(per[sel]):.0f}")
    gap = t[1:, 0] - t[:-1, 4]
    print(f"softmax warp 4: mean cycles wait_S {d[sel, 0].mean():.0f}  load+exchange {d[sel, 1].mean():.0f}  "
          f"exp+store {d[sel, 2].mean():.0f}  arrive(+epilogue) {d[sel, 3].mean():.0f}  gap {gap[sel].mean():.0f}  "
          f"period {per[sel].mean():.0f}")
    g_sel = gap[sel]
    print("gap histogram (cycles):", np.histogram(g_sel, bins=[0, 50, 100, 150, 200, 300, 400, 600, 1000, 10**6])[0].tolist(),
          "bins 0/50/100/150/200/300/400/600/1000/inf")
    big = np.argsort(-gap[sel])[:6] + 20
    print("largest gaps (block, gap, next wait_S):", [(int(i), int(gap[i]), int(d[i + 1, 0])) for i in big])
    dm = np.diff(m[:, :5], axis=1)
    perm = m[1:, 0] - m[:-1, 0]
    print(f"MMA: median cycles wait_P {np.median(dm[sel, 0]):.0f}  wait_V {np.median(dm[sel, 1]):.0f}  PV issue "
          f"{np.median(dm[sel, 2]):.0f}  S issue {np.median(dm[sel, 3]):.0f}  period {np.median(perm[sel]):.0f}")
    # slot 5 of block b: K_b ready inside the issue of S_b (which follows PV_{b-2}, slot 3 of b-2)
    kw = m[22:200, 5] - m[20:198, 3]
    print(f"MMA: median cycles from PV_(b-2) issued to K_b ready {np.median(kw):.0f}; S_b issue after K ready "
          f"{np.median(m[22:200, 4 - 4 + 4] * 0 + (m[20:198, 4] - m[22:200, 5])):.0f}")
    if "--raw" in sys.argv or os.environ.get("TRACE_RAW"):
        base = m[40, 0]
        print("blocks 40..60, cycles rel. to MMA slot 0 of block 40")
        print("MMA: [wait_P start, P ok, V ok, PV issued, S_(b+2) issued, K_(b) ready]  softmax warp 4: [start, S ok, "
              "exchanged, P stored, arrived]")
        for b in range(40, 60):
            print(b, [int(x - base) for x in m[b, :6]], [int(x - base) for x in t[b, :5]])
        arr = np.zeros((256, 8, 5), dtype=np.uint64)
        assert lib.attncache_debug_split_trace_arr(ctypes.c_void_p(arr.ctypes.data)) == 0
        a = arr.astype(np.int64)
        ph = np.diff(a, axis=2)  # S wait, load+exchange, exp+store, arrive
        print("per softmax warp 4..11, median cycles over blocks 20..200: [start rel. warp 4, S wait, load+exchange, "
              "exp+store, arrive]")
        for w in range(8):
            print(4 + w, int(np.median(a[20:200, w, 0] - a[20:200, 0, 0])),
                  np.median(ph[20:200, w], axis=0).astype(int).tolist())
        print("median MMA P-ok after last arrival:", int(np.median(m[20:200, 1] - a[20:200, :, 4].max(axis=1))))
    sys.exit(0)
buf = np.zeros((2, 256, 6), dtype=np.uint64)
assert lib.attncache_debug_att_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
t = buf.astype(np.int64)
for grp in range(2):
    d = np.diff(t[grp], axis=1)
    gap = t[grp, 1:, 0] - t[grp, :-1, 5]
    per = t[grp, 1:, 0] - t[grp, :-1, 0]
    sel = slice(20, 200)
    print(f"group {grp}: median cycles  wait_S {np.median(d[sel, 0]):.0f}  load_S {np.median(d[sel, 1]):.0f}  "
          f"max {np.median(d[sel, 2]):.0f}  exp+store {np.median(d[sel, 3]):.0f}  arrive {np.median(d[sel, 4]):.0f}  "
          f"gap {np.median(gap[sel]):.0f}  period {np.median(per[sel]):.0f}")
print("first blocks of group 0 (wait, load, max, exp, arrive, gap):")
for i in range(20, 30):
    print(list(np.diff(t[0, i])), t[0, i + 1, 0] - t[0, i, 5])
mm = np.zeros((512, 8), dtype=np.uint64)
assert lib.attncache_debug_att_trace_mma(ctypes.c_void_p(mm.ctypes.data)) == 0
m = mm.astype(np.int64)
print("MMA warp, events 40..60 (cycles rel. to event 40 start): start, k_ready, S_issued | pv: start, p_full, v_full, issued")
base = m[40, 0]
for e in range(40, 60):
    print(e, [int(x - base) if x else None for x in m[e, :7]])
