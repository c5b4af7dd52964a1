"""Timeline of the capture kernel (f1) at a config's shape: builds the library with -DCAP_TRACE out of tree, runs
the capture of `rows` prefills once and prints, per epilogue warp (4-7 group 0, 8-11 group 1; lane 0 of CTA 0),
the median cycles of each block-pass phase: S wait, TMEM load of S, the body (pass 0: max + exp + sum; pass 1:
exp + pack + stores), and the per-block-pass period, split by pass.
Usage: python scripts/capture_trace.py [config] [rows]"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
env = dict(os.environ, ATTNCACHE_BUILD_ROOT="/tmp/captrace", ATTNCACHE_EXTRA_FLAGS="-DCAP_TRACE " + os.environ.get("TRACE_FLAGS", ""))
subprocess.check_call([sys.executable, "-m", "paper_2510_25979_b200.build"], env=env, cwd=ROOT, stdout=subprocess.DEVNULL)
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
ac.lib_path = "/tmp/captrace/lib/libattncache.so"
name = sys.argv[1] if len(sys.argv) > 1 else "long_prefill"
cfg = synth.CONFIGS[name]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B - cfg.n_hit
ctx = ac.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
Q, K = (torch.randn(rows, cfg.L, cfg.H, cfg.S, cfg.d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
out = ac.attncache_capture_maps(ctx, Q, K)
torch.cuda.synchronize()
ac.attncache_capture_maps(ctx, Q, K, out=out)
torch.cuda.synchronize()
lib = ac.load_library()
buf = np.zeros((8, 512, 4), dtype=np.uint64)
assert lib.attncache_debug_cap_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
t = buf.astype(np.int64)
sel = slice(20, 500)
for w in range(8):
    d = np.diff(t[w, sel], axis=1)
    per = np.diff(t[w, sel, 0])
    print(f"warp {4 + w}: median S wait {np.median(d[:, 0]):.0f}  load {np.median(d[:, 1]):.0f}  body "
          f"{np.median(d[:, 2]):.0f}  (body p10/p90 {np.percentile(d[:, 2], 10):.0f}/{np.percentile(d[:, 2], 90):.0f})"
          f"  period {np.median(per):.0f}  mean period {per.mean():.0f}")
# bodies split in two clusters: pass 0 (max + exp + sum) vs pass 1 (exp + stores)
d = np.diff(t[0, sel], axis=1)
print("warp 4 block-passes 40..60: [S wait, load, body, gap to next]")
for i in range(40, 60):
    print(i, [int(x) for x in np.diff(t[0, i])], int(t[0, i + 1, 0] - t[0, i, 3]))
