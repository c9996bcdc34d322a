O=gpurun_out
python scripts/profile_solve.py C4 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_twist_lane_dd|k_fixed_chunk|k_rqi2|k_fixed_step" -s 0 -c 12 \
    -o /tmp/s14_c4 python scripts/profile_solve.py C4 1 > $O/s14.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/s14_c4.ncu-rep $O/s14_c4.json C4 > /dev/null 2>&1; echo "sum rc=$?"
ncu -i /tmp/s14_c4.ncu-rep --page details --csv > $O/s14_details.csv 2>&1
