O=gpurun_out
python scripts/sweep_env.py C3 2 ""
python scripts/sweep_env.py C4 2 ""
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sd.py tests/test_gpu_families.py -q -x > $O/s16_tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/s16_tests.log
