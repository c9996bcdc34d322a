O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s8_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/s8_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > $O/s8_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s8_pytest.log
python bench.py > $O/s8_bench_C2.json 2> $O/s8_bench_C2.err; echo "bench rc=$?"; cat $O/s8_bench_C2.json | head -c 600; echo
