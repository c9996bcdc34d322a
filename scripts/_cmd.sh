O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for w in C2 C5a C4; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload $w | python scripts/bench_summary.py $w; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv python scripts/profile_solve.py C2 2 > /dev/null 2>&1; python scripts/launch_summary.py $O/launches_C2.csv 2>/dev/null | grep -E "pick2|fixed_step|build_q|launches,"
