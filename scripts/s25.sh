O=gpurun_out
timeout 300 python scripts/sweep_env.py C2 5 "" 2>&1 | tail -1
timeout 300 python scripts/sweep_env.py C5b 3 "" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_zwrite" --csv --log-file $O/s25_z.csv python scripts/profile_solve.py C2 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_support.py tests/test_gpu_parity.py -q -x -k "support or config_full or small" > $O/s25_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/s25_tests.log
