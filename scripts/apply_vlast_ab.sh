#!/bin/bash
# Paired A.V: V of a unit's last pair loaded evict_first (last use) vs evict_last throughout (out-of-tree builds;
# configs[3] and configs[2] A.V timings, then ncu DRAM bytes of one configs[3] launch per variant).
mkdir -p gpurun_out
for v in "prod:" "vlast:-DAPPLY_VLAST"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/app_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1
done
for r in 1 2 3; do
  for n in prod vlast; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so python scripts/apply_bench.py long_prefill 16 16 20) | $(ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so python scripts/apply_bench.py llama3_8b 115 128 10)"
  done
done
for n in prod vlast; do
  ATTNCACHE_LIB=/tmp/app_$n/lib/libattncache.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k "regex:apply_pair" -s 3 -c 1 python scripts/apply_bench.py long_prefill 16 16 1 2>&1 | \
    grep -E "dram__bytes|gpu__time" | sed "s/^/$n /"
done
