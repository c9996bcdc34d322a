O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload C2 | python scripts/bench_summary.py C2
