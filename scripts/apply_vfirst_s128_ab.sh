#!/bin/bash
# Single-row-block A.V (S <= 128, configs[1]): V loaded evict_first (read once) vs evict_last (APPLY_EXP=3),
# out-of-tree builds; A.V timings at configs[1] and the bench step.
mkdir -p gpurun_out
for v in "prod:" "vfirst:-DAPPLY_EXP=3"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/app_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1 || echo "build $n failed"
done
for r in 1 2 3; do
  for n in prod vfirst; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so python scripts/apply_bench.py llama32_1b 205 256 20)"
  done
done
