#!/bin/bash
# World-1 pipelined step (bench.py --force-dist): side streams (next batch's search / placement, relocation) at
# high priority (-1, bench default) vs normal priority (0), interleaved, REPS rounds; single-GPU step beside.
mkdir -p gpurun_out
CFG=${CFG:-llama32_1b}
for r in $(seq ${REPS:-3}); do
  echo "single: $(python bench.py --config $CFG --steps 30 --warmup 3 --no-cpu-baseline --no-search-sweep --no-target 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')"
  for p in ${PRIOS:--1 0}; do
    echo "prio $p: $(ATTNCACHE_BENCH_SIDE_PRIORITY=$p python bench.py --config $CFG --steps 30 --warmup 3 --force-dist --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d.get("other_scaling", {}).get("ms_per_step"))')"
  done
done
