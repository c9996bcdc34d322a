python scripts/sweep_env.py C3 3 ""
python scripts/sweep_env.py C4 2 ""
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_build_q" --csv --log-file gpurun_out/s18_bq.csv python scripts/profile_solve.py C3 1 > /dev/null 2>&1; grep k_build_q gpurun_out/s18_bq.csv | cut -c1-200
