#!/bin/bash
# One GPU session: build, full GPU test suite, smoke, the default bench line, and configs 2/3 bench lines.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build-failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1=$?
for c in llama3_8b long_prefill; do
  timeout 900 python bench.py --config $c --no-search-sweep --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
done
python scripts/bench_summary.py < gpurun_out/bench_c1.json 2>/dev/null | head -30
