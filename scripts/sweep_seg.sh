for cfg in "16 8 128" "16 16 128" "16 32 96" "16 16 192" "8 16 128" "32 16 128"; do
  set -- $cfg
  MRRR_TARGET_CHAINS=$(( $1 * 1024 )) MRRR_SEGK=$2 MRRR_SEGW=$3 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --workload C2 | python scripts/bench_summary.py "C2 tc=${1}K K=$2 W=$3"
done
for w in C5a C5b C1; do MRRR_TARGET_CHAINS=16384 MRRR_SEGK=16 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 --workload $w | python scripts/bench_summary.py "$w tc16K K16"; done
