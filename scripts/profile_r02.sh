#!/bin/bash
# Round-2 ncu evidence (B200_PROFILING.md recipe; every profiled command first runs plain and exits 0):
#   * the bench's launch list (gpu__time_duration, --clock-control none);
#   * --set full of the search kernel at configs[4] B = 1024 and 8192 (tensor-pipe utilisation);
#   * --set full of the hot kernels of the bench step (configs[1]) and of A.V / attention at configs[2] / [3].
set -u
P=${1:-r02a}
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-search-sweep --no-target"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
$B > gpurun_out/plain_c1.log 2>&1 && echo plain_c1=ok &&
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function \
    -k "regex:^(search_|keys_|select_|apply_|attend|capture_|linear_|normalize_|rope|copy_rows|route_)" -c 3000 \
    --csv --log-file gpurun_out/${P}_launches.csv $B > /dev/null 2>&1; echo launches=$?
for b in 1024 8192; do
  python scripts/search_bench.py $b 2 > gpurun_out/plain_search_$b.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:search_tc" -s 2 -c 1 -o gpurun_out/${P}_search_$b \
      python scripts/search_bench.py $b 1 > gpurun_out/ncu_search_$b.log 2>&1; echo search_$b=$?
done
ncu --set full --clock-control none --import-source on -k "regex:apply_tc|apply_pair|attend_tc|attend_split|search_tc" -s 8 -c 6 \
    -o gpurun_out/${P}_full_c1 $B > gpurun_out/ncu_full_c1.log 2>&1; echo full_c1=$?
python scripts/apply_bench.py llama3_8b 115 128 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:apply_tc|apply_pair" -s 3 -c 1 -o gpurun_out/${P}_apply_llama3_8b \
    python scripts/apply_bench.py llama3_8b 115 128 1 > gpurun_out/ncu_apply_c2.log 2>&1; echo apply_c2=$?
for c in "long_prefill 16" "llama3_8b 13"; do
  set -- $c
  python scripts/attend_bench.py $1 $2 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:attend_(tc|split)" -s 3 -c 1 -o gpurun_out/${P}_attend_$1 \
      python scripts/attend_bench.py $1 $2 1 > gpurun_out/ncu_attend_$1.log 2>&1; echo attend_$1=$?
done
python scripts/capture_bench.py long_prefill 16 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:capture_tc" -s 3 -c 1 -o gpurun_out/${P}_capture_long_prefill \
    python scripts/capture_bench.py long_prefill 16 > gpurun_out/ncu_capture.log 2>&1; echo capture=$?
ls -la gpurun_out/ | grep ${P}
