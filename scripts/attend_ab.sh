#!/bin/bash
# A/B of compile-time variants of the attention kernels: VARIANTS="name:flags ..." (flags comma-separated),
# each built out of tree and timed on configs[3] / [2] misses and configs[1] misses (d = 64).
for v in ${VARIANTS:-base:}; do
  n=${v%%:*}; f=${v#*:}; f=${f//,/ }
  ATTNCACHE_BUILD_ROOT=/tmp/ab_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null || { echo "$n build failed"; continue; }
  L=/tmp/ab_$n/lib/libattncache.so
  IFS=";" read -ra cases <<< "${CASES:-long_prefill 16;llama3_8b 13;llama32_1b 51}"
  for c in "${cases[@]}"; do
    set -- $c
    echo "$n: $(ATTNCACHE_LIB=$L timeout 120 python scripts/attend_bench.py $1 $2 ${REPS:-10} | tail -1)"
  done
done
