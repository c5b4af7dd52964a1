#!/bin/bash
# Sweeps the number of polynomial-exp2 key pairs per 8 (SPLIT_POLY, the d=128 split kernel) on configs[3]/[2] attention.
for n in ${PAIRS:-0 2 3 4}; do
  ATTNCACHE_BUILD_ROOT=/tmp/poly$n ATTNCACHE_EXTRA_FLAGS="-DSPLIT_POLY=$n" python -m paper_2510_25979_b200.build > /dev/null
  echo "POLY=$n: $(ATTNCACHE_LIB=/tmp/poly$n/lib/libattncache.so python scripts/attend_bench.py long_prefill 16 10) | $(ATTNCACHE_LIB=/tmp/poly$n/lib/libattncache.so python scripts/attend_bench.py llama3_8b 13 10)"
done
