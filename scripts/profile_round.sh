#!/bin/bash
# ncu evidence for profiles/: the bench's launch list, --set full captures of the hot kernels at configs[1]
# (the bench workload) and of the d=128 attention at configs[2]/[3].  Each profiled command first runs
# plain and must exit 0 (B200_PROFILING.md).
set -u
P=${1:-r01b}
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-search-sweep"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
$B > gpurun_out/plain_c1.log 2>&1 && echo plain_c1=ok &&
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function \
    -k "regex:^(search_|keys_|select_|apply_|attend|capture_|linear_|normalize_|rope|copy_rows|route_)" -c 3000 \
    --csv --log-file gpurun_out/${P}_launches.csv $B > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k "regex:apply_tc|attend_tc|search_tc|linear_tc|keys_decode|capture_tc" -s 8 -c 8 \
    -o gpurun_out/${P}_full_c1 $B > gpurun_out/ncu_full_c1.log 2>&1; echo full_c1=$?
for c in "long_prefill 16" "llama3_8b 13"; do
  set -- $c
  python scripts/attend_bench.py $1 $2 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:attend_(tc|split)" -s 3 -c 1 -o gpurun_out/${P}_attend_$1 \
      python scripts/attend_bench.py $1 $2 1 > gpurun_out/ncu_attend_$1.log 2>&1; echo attend_$1=$?
done
python scripts/capture_bench.py llama32_1b 51 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:capture_tc" -s 3 -c 1 -o gpurun_out/${P}_capture_c1 \
    python scripts/capture_bench.py llama32_1b 51 > gpurun_out/ncu_capture.log 2>&1; echo capture=$?
