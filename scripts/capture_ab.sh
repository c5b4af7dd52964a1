#!/bin/bash
# A/B of capture-kernel compile-time variants: VARIANTS="name:flags ..." (flags comma-separated), each built
# out of tree and timed on configs[1] / [2] / [3] misses (packed bf16 maps).
for v in ${VARIANTS:-base:}; do
  n=${v%%:*}; f=${v#*:}; f=${f//,/ }
  ATTNCACHE_BUILD_ROOT=/tmp/cab_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null || { echo "$n build failed"; continue; }
  IFS=";" read -ra cases <<< "${CASES:-llama32_1b 51;llama3_8b 13;long_prefill 16}"
  for c in "${cases[@]}"; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/cab_$n/lib/libattncache.so timeout 120 python scripts/capture_bench.py $c | tail -1)"
  done
done
