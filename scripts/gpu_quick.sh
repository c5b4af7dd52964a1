#!/bin/bash
# quick GPU check: parity tests (optionally filtered) + bench summary line
K=${1:-""}
if [ -n "$K" ]; then timeout 400 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 200 -k "$K" > gpurun_out/pytest_q.log 2>&1;
else timeout 400 python -m pytest tests/test_gpu_parity.py -q -rf -x --timeout 200 > gpurun_out/pytest_q.log 2>&1; fi
echo pytest_exit=$?; tail -3 gpurun_out/pytest_q.log | cut -c1-600
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('tok/s %.4g ms %.4f search %.4f apply %.4f (frac %.3f) attend %.4f (hbm %.3f) full %.4f speedup %.3f' % (d['value'], d['ms_per_step'], d['stages']['search']['ms'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['stages']['attend_full_misses']['ms'], d['stages']['attend_full_misses']['hbm_frac'], d['speedup_vs_full_attention']['full_attention_ms'], d['speedup_vs_full_attention']['batch']))"
