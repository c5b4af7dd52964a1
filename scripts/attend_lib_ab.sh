for L in ab_old/lib/libattncache.so paper_2510_25979_b200/lib/libattncache.so ab_old/lib/libattncache.so paper_2510_25979_b200/lib/libattncache.so; do
  for c in "llama32_1b 51" "llama3_8b 13" "long_prefill 16"; do
    echo "$L $c: $(ATTNCACHE_LIB=$L python scripts/attend_bench.py $c 20 | tail -1)"
  done
done
