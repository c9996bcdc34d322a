O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for w in C2 C5a; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload $w | python scripts/bench_summary.py $w; done
