O=gpurun_out
timeout 300 python scripts/sweep_env.py C3 3 "" 2>&1 | tail -1
timeout 300 python scripts/sweep_env.py C4 2 "" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_clu_build_seg" --csv --log-file $O/s24_b.csv python scripts/profile_solve.py C3 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "C3 or C4 or wilk or glued" > $O/s24_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/s24_tests.log
