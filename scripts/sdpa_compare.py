"""External sanity point for the miss path: torch SDPA (cuDNN / flash backends, library
code, not this repo's path) on the same causal shapes as scripts/attend_bench.py."""
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

for name, rows, L, H, S, d in (("long_prefill", 16, 8, 32, 1024, 128), ("llama3_8b", 13, 32, 32, 256, 128),
                               ("llama32_1b", 51, 16, 32, 128, 64)):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(rows * L, H, S, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    flops = rows * L * H * 4.0 * d * S * (S + 1) / 2
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([be]):
                for _ in range(3):
                    F.scaled_dot_product_attention(q, k, v, is_causal=True)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    F.scaled_dot_product_attention(q, k, v, is_causal=True)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                print(f"{name} {be.name}: {ms:.3f} ms {flops / ms / 1e9:.1f} TFLOP/s")
        except Exception as ex:  # noqa: BLE001
            print(f"{name} {be.name}: unavailable ({str(ex)[:80]})")
    sys.stdout.flush()
