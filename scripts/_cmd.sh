O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for v in 0 10000 1073741824; do
MRRR_SEGCH2=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload C2 | python scripts/bench_summary.py C2 CH2=$v
MRRR_SEGCH2=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2 --workload C5a | python scripts/bench_summary.py C5a CH2=$v
done
for tc in 24576 32768; do MRRR_TARGET_CHAINS=$tc timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload C2 | python scripts/bench_summary.py C2 CH2all TC=$tc; done
