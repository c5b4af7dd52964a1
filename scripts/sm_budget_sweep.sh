#!/bin/bash
# World-1 pipelined multi-GPU step (bench.py --force-dist) against the single-GPU step, for several SM budgets
# of the side streams (--aux-sms; attncache_ctx_set_sm_budget).  REPS runs each, median printed by the caller.
mkdir -p gpurun_out
CFG=${CFG:-llama32_1b}
for r in $(seq ${REPS:-3}); do
  echo "single: $(python bench.py --config $CFG --steps 30 --warmup 3 --no-cpu-baseline --no-search-sweep --no-target 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')"
  for a in ${AUX:-0 4 8 16}; do
    echo "aux $a: $(python bench.py --config $CFG --steps 30 --warmup 3 --force-dist --aux-sms $a --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d.get("other_scaling", {}).get("ms_per_step"))')"
  done
done
