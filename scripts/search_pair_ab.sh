#!/bin/bash
# two-query-tile search kernel vs the one-tile kernel at configs[4] (B = 1024, 8192) and a mid batch
for v in "pair:" "single:-DSEARCH_NO_PAIR"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/sp_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1
  for b in 256 1024 8192; do echo "$n: $(ATTNCACHE_LIB=/tmp/sp_$n/lib/libattncache.so python scripts/search_bench.py $b 5)"; done
done
