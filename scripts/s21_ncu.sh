O=gpurun_out
python scripts/profile_solve.py C3 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_clu_build_seg|k_clu_attempt_seg|k_rqi2" -s 0 -c 4 \
    -o /tmp/s21 python scripts/profile_solve.py C3 1 > $O/s21.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/s21.ncu-rep $O/s21.json C3 > /dev/null 2>&1
ncu -i /tmp/s21.ncu-rep --page details --csv > $O/s21_details.csv 2>&1
ncu -i /tmp/s21.ncu-rep --page source --csv --print-source sass -k regex:"k_clu_build_seg" > $O/s21_src_build.csv 2>&1
