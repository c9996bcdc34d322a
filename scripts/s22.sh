O=gpurun_out
python scripts/sweep_env.py C3 3 ""
python scripts/sweep_env.py C4 2 ""
timeout 1700 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_families.py tests/test_gpu_sd.py -q -x > $O/s22_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/s22_tests.log
