O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/s1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x --durations=25 > $O/s1_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 $O/s1_pytest.log
python bench.py > $O/s1_bench_C2.json 2> $O/s1_bench_C2.err; echo "bench rc=$?"; cat $O/s1_bench_C2.json
python bench.py --early-stop > $O/s1_bench_C2_es.json 2> $O/s1_bench_C2_es.err; echo "bench es rc=$?"; cat $O/s1_bench_C2_es.json
