#!/bin/bash
# A/B of compile-time variants of the capture kernel: VARIANTS="name:flags ..." (flags comma-separated), each built
# out of tree and timed at configs 1 / 2 / 3 (scripts/capture_bench.py).
for v in ${VARIANTS:-base:}; do
  n=${v%%:*}; f=${v#*:}; f=${f//,/ }
  ATTNCACHE_BUILD_ROOT=/tmp/cab_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null || { echo "$n build failed"; continue; }
  for c in ${CASES:-llama32_1b llama3_8b long_prefill}; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/cab_$n/lib/libattncache.so timeout 120 python scripts/capture_bench.py $c | tail -1)"
  done
done
