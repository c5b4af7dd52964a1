#!/bin/bash
# A.V kernel variants (-DAPPLY_EXP=n): 0 product (maps: normal L2 policy), 1 maps with evict_first, 2 V with the normal policy.
for n in ${EXPS:-0 1 2}; do
  ATTNCACHE_BUILD_ROOT=/tmp/apexp$n ATTNCACHE_EXTRA_FLAGS="-DAPPLY_EXP=$n" python -m paper_2510_25979_b200.build > /dev/null
  echo "APPLY_EXP=$n: $(ATTNCACHE_LIB=/tmp/apexp$n/lib/libattncache.so python scripts/apply_bench.py llama3_8b 115 128 10) | $(ATTNCACHE_LIB=/tmp/apexp$n/lib/libattncache.so python scripts/apply_bench.py llama32_1b 205 256 20)"
done
