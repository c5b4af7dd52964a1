#!/bin/bash
# configs[4] search: the CTA-pair kernel (scripts/experiments/search_cta2_kernel.cu.txt, copied into
# kernels_tc_search.cu; default for B >= 512 there) against the one-CTA kernel (-DSEARCH_NO_PAIR).
ATTNCACHE_BUILD_ROOT=/tmp/snp ATTNCACHE_EXTRA_FLAGS="-DSEARCH_NO_PAIR" python -m paper_2510_25979_b200.build > /dev/null || exit 1
for B in ${BATCHES:-512 1024 2048 8192}; do
  echo "pair   $(timeout 120 python scripts/search_bench.py $B 10)"
  echo "single $(ATTNCACHE_LIB=/tmp/snp/lib/libattncache.so timeout 120 python scripts/search_bench.py $B 10)"
done
