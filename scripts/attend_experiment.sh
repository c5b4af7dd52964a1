#!/bin/bash
# Builds experiment variants of the library (-DATT_EXP=n) out of tree and times attention on each.
# 0 = product kernel, 1 = softmax math skipped, 2 = exp2 replaced by a multiply (no MUFU), 3 = no Q/K/V loads.
cfg=${1:-long_prefill}; rows=${2:-16}
for n in ${EXPS:-0 1 2 3}; do
  ATTNCACHE_BUILD_ROOT=/tmp/attexp$n ATTNCACHE_EXTRA_FLAGS="-DATT_EXP=$n" python -m paper_2510_25979_b200.build > /dev/null
  echo "ATT_EXP=$n: $(ATTNCACHE_LIB=/tmp/attexp$n/lib/libattncache.so python scripts/attend_bench.py $cfg $rows 10)"
done
