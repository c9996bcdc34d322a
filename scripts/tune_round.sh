#!/bin/bash
# bench a workload under several environment settings (developer sweep)
#   VAR=MRRR_TARGET_CHAINS VALS="24576 65536" WL=C2 bash scripts/tune_round.sh
VAR=${VAR:-MRRR_TARGET_CHAINS}
for v in ${VALS:-24576 40960 65536 131072}; do
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps ${STEPS:-3} --warmup 2 --workload ${WL:-C2} \
    | python scripts/bench_summary.py "$WL $VAR=$v"
done
