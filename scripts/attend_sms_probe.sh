#!/bin/bash
# Is the d = 128 attention power-limited?  The same launch on fewer SMs (-DSM_EXPERIMENT, AC_ATTEND_SMS): if the
# per-SM rate rises as SMs are taken away, the clock had headroom only under a lower total power.
ATTNCACHE_BUILD_ROOT=/tmp/smx ATTNCACHE_EXTRA_FLAGS="-DSM_EXPERIMENT" python -m paper_2510_25979_b200.build > /dev/null || exit 1
for n in 148 128 111 96 74; do
  echo "sms $n: $(AC_ATTEND_SMS=$n ATTNCACHE_LIB=/tmp/smx/lib/libattncache.so python scripts/attend_bench.py long_prefill 16 10 | tail -1)"
done
