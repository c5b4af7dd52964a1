for v in "pair:" "nopair:-DAPPLY_NO_PAIR"; do
  n=${v%%:*}; f=${v#*:}
  ATTNCACHE_BUILD_ROOT=/tmp/apv_$n ATTNCACHE_EXTRA_FLAGS="$f" python -m paper_2510_25979_b200.build > /dev/null 2>&1
  for c in "long_prefill 16 32" "llama3_8b 115 128" "llama32_1b 205 256"; do
    echo "$n: $(ATTNCACHE_LIB=/tmp/apv_$n/lib/libattncache.so python scripts/apply_bench.py $c 10)"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply or partial or full_step or repeat or virtual or gqa or noncausal or capture_then or host_prefill or collective" 2>&1 | tail -3
