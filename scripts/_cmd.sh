O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for v in 0 1; do for kw in "8 192" "4 192"; do set -- $kw
MRRR_RQIBULK=$v MRRR_RQISEGK=$1 MRRR_RQISEGW=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 --workload C2 | python scripts/bench_summary.py C2 bulk=$v K=$1 W=$2
MRRR_RQIBULK=$v MRRR_RQISEGK=$1 MRRR_RQISEGW=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2 --workload C5a | python scripts/bench_summary.py C5a bulk=$v K=$1 W=$2
done; done
timeout 900 ncu --clock-control none -k regex:"k_fixed_chunk" -s 2 -c 2 --csv --metrics gpu__time_duration.sum,smsp__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_write.sum python scripts/profile_solve.py C2 2 > $O/ncu_m.csv 2>&1; echo rc=$?
