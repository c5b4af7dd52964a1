#!/bin/bash
# The d = 128 miss attention at configs[3] / configs[2] shapes against torch SDPA's cuDNN backend (library code),
# interleaved on one box (both are power-capped at S = 1024, so alternating runs keep the comparison fair).
for r in 1 2 3; do
  python scripts/attend_bench.py long_prefill 16 20 2>&1 | tail -1
  python scripts/sdpa_compare.py 2>&1 | grep -E "CUDNN" | head -2
  python scripts/attend_bench.py llama3_8b 13 20 2>&1 | tail -1
done
