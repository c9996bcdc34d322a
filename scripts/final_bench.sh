#!/bin/bash
# round-end numbers: default bench (C2) + every config + the reference (oracle) arm
O=gpurun_out
timeout 900 python bench.py > $O/final_bench_C2.log 2>&1; echo "bench C2 rc=$?"; tail -1 $O/final_bench_C2.log | cut -c1-200
for w in C1 C3 C4 C5b C5a; do
  timeout 1200 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/final_bench_$w.log 2>&1; echo "bench $w rc=$?"
  python scripts/bench_summary.py $w < $O/final_bench_$w.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/final_reference_C2.log 2>&1; echo "reference rc=$?"; tail -1 $O/final_reference_C2.log | cut -c1-300
