#!/bin/bash
# A.V kernel variants at configs[1] / [2] shapes (ATTNCACHE_EXTRA_FLAGS builds out of tree).
for v in ${VARIANTS:-"prod:" "oldload:-DAPPLY_OLD_LOADER" "oldall:-DAPPLY_OLD_LOADER -DAPPLY_V2D -DAPPLY_O2D"}; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/apv_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1
  echo "$n: $(ATTNCACHE_LIB=/tmp/apv_$n/lib/libattncache.so python scripts/apply_bench.py llama32_1b 205 256 20) | $(ATTNCACHE_LIB=/tmp/apv_$n/lib/libattncache.so python scripts/apply_bench.py llama3_8b 115 128 10)"
done
