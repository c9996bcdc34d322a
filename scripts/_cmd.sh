O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for v in 16 8 4 2; do MRRR_DEVFRAC=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 7 --warmup 3 --workload C2 | python scripts/bench_summary.py C2 DEVFRAC=$v; done
for v in 16 4; do MRRR_DEVFRAC=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --workload C5b | python scripts/bench_summary.py C5b DEVFRAC=$v; done
