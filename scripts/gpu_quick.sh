#!/bin/bash
# quick GPU check: parity tests (optionally filtered by -k) + one bench line summary
K=${1:-""}
if [ -n "$K" ]; then timeout 400 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 200 -k "$K" > gpurun_out/pytest_q.log 2>&1;
else timeout 400 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 200 > gpurun_out/pytest_q.log 2>&1; fi
echo pytest_exit=$?; tail -2 gpurun_out/pytest_q.log | cut -c1-600
shift
timeout 600 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench.log 2>&1; echo bench=$?
python scripts/bench_summary.py < gpurun_out/bench.log
