O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for kw in "1 128" "8 128" "8 256" "4 256"; do set -- $kw
for w in C3 C4; do MRRR_SEGXK=$1 MRRR_SEGXW=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 --workload $w | python scripts/bench_summary.py $w K=$1 W=$2; done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python scripts/profile_solve.py C3 1 > /dev/null 2>&1; python scripts/launch_summary.py $O/launches_C3.csv 2>/dev/null | head -8
