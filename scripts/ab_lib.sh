set -x
B="python bench.py --steps 30 --warmup 3 --no-target --no-search-sweep --no-cpu-baseline"
cp paper_2510_25979_b200/lib/libattncache.so /tmp/new.so
for i in 1 2; do
$B > gpurun_out/ab_new_$i.log 2>&1
cp ab_old/lib/libattncache.so paper_2510_25979_b200/lib/libattncache.so
$B > gpurun_out/ab_old_$i.log 2>&1
cp /tmp/new.so paper_2510_25979_b200/lib/libattncache.so
done
for f in gpurun_out/ab_*.log; do echo $f; python scripts/bench_summary.py < $f | head -1; done
