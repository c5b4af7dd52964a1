#!/bin/bash
# d = 128 split attention: L2 policies of its TMA loads (ATT2_POL: 1 = Q evict_first, 2 = also K/V evict_last)
# against the default (all evict_normal); out-of-tree builds, configs[3] and configs[2] misses, then ncu DRAM bytes.
mkdir -p gpurun_out
for v in "prod:" "q1:-DATT2_POL=1" "q2:-DATT2_POL=2"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/att_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1 || echo "build $n failed"
done
for r in 1 2 3; do
  for n in prod q1 q2; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/att_$n/lib/libattncache.so python scripts/attend_bench.py long_prefill 16 20 2>&1 | tail -1) | $(ATTNCACHE_LIB=/tmp/att_$n/lib/libattncache.so python scripts/attend_bench.py llama3_8b 13 20 2>&1 | tail -1)"
  done
done
for n in prod q1 q2; do
  ATTNCACHE_LIB=/tmp/att_$n/lib/libattncache.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k "regex:attend_split" -s 3 -c 1 python scripts/attend_bench.py long_prefill 16 1 2>&1 | \
    grep -E "dram__bytes|gpu__time" | sed "s/^/$n /"
done
