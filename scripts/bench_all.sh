#!/bin/bash
# bench lines for every BASELINE configuration (C2 is bench.py's default workload) + launch lists of C3/C4
O=gpurun_out
for w in C1 C2 C3 C4 C5b C5a; do
  st=5; [ $w = C5a ] && st=3
  python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/r02_bench_$w.json 2> $O/r02_bench_$w.err; echo "$w rc=$?"
done
python scripts/subset_sweep.py C2 C5a > $O/r02_subset_sweep.txt 2>&1; echo "subset rc=$?"
for w in C3 C4; do
  python scripts/profile_solve.py $w 2 > $O/r02_plain_$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_$w.csv \
      python scripts/profile_solve.py $w 2 > /dev/null 2>&1; echo "launches $w rc=$?"
done
