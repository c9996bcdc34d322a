#!/bin/bash
# round-2 closing evidence: smoke, GPU suite, bench lines of every configuration, launch lists C2/C3/C4
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/r02d_smoke.log
timeout 1800 python -m pytest tests -q -m gpu > $O/r02d_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02d_pytest.log
python bench.py > $O/r02d_bench_C2.json 2> $O/r02d_bench_C2.err; echo "bench C2 rc=$?"
for w in C1 C3 C4 C5b C5a; do
  st=5; [ $w = C5a ] && st=3
  python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/r02d_bench_$w.json 2> $O/r02d_bench_$w.err; echo "$w rc=$?"
done
for w in sd; do python bench.py --profile sd --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02d_bench_sd_C2.json 2> /dev/null; echo "sd rc=$?"; done
python bench.py --early-stop --no-cpu-baseline > $O/r02d_bench_es_C2.json 2> /dev/null; echo "es rc=$?"
for w in C2 C3 C4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02d_launches_$w.csv \
      python scripts/profile_solve.py $w 2 > /dev/null 2>&1; echo "launch list $w rc=$?"
done
