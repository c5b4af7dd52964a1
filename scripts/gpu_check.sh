#!/bin/bash
# GPU round check: smoke, the -m gpu suite, the default bench line, the world-1 collective bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -rfs --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_all.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_all.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench=$?
tail -c 600 gpurun_out/bench.err
timeout 600 python bench.py --steps 20 --warmup 3 --force-dist > gpurun_out/bench_dist.log 2>gpurun_out/bench_dist.err; echo bench_dist=$?
tail -c 600 gpurun_out/bench_dist.err
fi
