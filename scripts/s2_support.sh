O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_support.py -q -x -s > $O/s2_support.log 2>&1; echo "support rc=$?"; tail -15 $O/s2_support.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sd.py -q -x > $O/s2_parity.log 2>&1; echo "parity rc=$?"; tail -3 $O/s2_parity.log
python bench.py > $O/s2_bench_C2.json 2> $O/s2_bench_C2.err; echo "bench rc=$?"; python -c "import json;j=json.load(open('$O/s2_bench_C2.json'));print(j['ms_per_step'],j['phases_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s2_launches_C2.csv python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "launch rc=$?"
python scripts/launch_summary.py $O/s2_launches_C2.csv 2>&1 | head -12
