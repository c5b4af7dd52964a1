#!/bin/bash
# d = 64 attention: Q / K / V slots per group (ATT_DEPTH 1 = one each, 2 = two each, 225.5 KB of shared memory),
# out-of-tree builds, configs[1]'s 51 misses (S = 128) and a longer-S d = 64 case.
for v in "d1:" "d2:-DATT_DEPTH=2"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/att_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1 || echo "build $n failed"
done
for r in 1 2 3; do
  for n in d1 d2; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/att_$n/lib/libattncache.so python scripts/attend_bench.py llama32_1b 51 20 2>&1 | tail -1)"
  done
done
