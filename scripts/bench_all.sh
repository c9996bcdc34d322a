#!/bin/bash
# bench lines for every BASELINE configuration (C2 is bench.py's default workload) + the single/double lines
O=gpurun_out
for w in C1 C2 C3 C4 C5b C5a; do
  st=5; [ $w = C5a ] && st=3
  python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/r02_bench_$w.json 2> $O/r02_bench_$w.err; echo "$w rc=$?"
done
for w in C1 C2; do
  python bench.py --profile sd --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02_bench_sd_$w.json 2> $O/r02_bench_sd_$w.err; echo "sd $w rc=$?"
done
