#!/bin/bash
# L2 cache-policy variants of the paired A.V kernel (configs[3] and configs[2] shapes; out-of-tree builds).
# (The APPLY_O_EVICT_FIRST / APPLY_MAP_EVICT_FIRST knobs were removed after this A/B; rebuild them
# from the tma_store_3d_hint / createpolicy lines described there to repeat it.)
for v in ${VARIANTS:-"prod:" "ofirst:-DAPPLY_O_EVICT_FIRST" "mfirst:-DAPPLY_MAP_EVICT_FIRST" "both:-DAPPLY_O_EVICT_FIRST -DAPPLY_MAP_EVICT_FIRST"}; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/app_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1
  for r in 1 2; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so python scripts/apply_bench.py long_prefill 16 16 20) | $(ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so python scripts/apply_bench.py llama3_8b 115 128 10)"
  done
done
