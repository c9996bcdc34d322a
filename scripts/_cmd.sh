O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
./scripts/fp64_peak
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for kw in "3 192" "4 192" "6 192" "8 192" "6 128"; do set -- $kw
MRRR_RQISEGK=$1 MRRR_RQISEGW=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload C2 | python scripts/bench_summary.py C2 K=$1 W=$2
MRRR_RQISEGK=$1 MRRR_RQISEGW=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2 --workload C5a | python scripts/bench_summary.py C5a K=$1 W=$2
done
