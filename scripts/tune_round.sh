#!/bin/bash
# bench C2 under several bisection chain budgets (developer sweep)
for tc in ${TCS:-24576 40960 65536 131072}; do
  echo "target_chains=$tc"
  MRRR_TARGET_CHAINS=$tc timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 ${BENCH_ARGS} | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=l['phases_ms']; print('  ms/step %.3f bis %.3f rqi %.3f root %.3f rounds %d negx %d' % (l['ms_per_step'], p['root_bisection'], p['singletons'], p['split_root'], l['stats']['rounds'], l['stats']['negcount_x']))"
done
