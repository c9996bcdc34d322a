O=gpurun_out
python scripts/profile_solve.py C3 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_rqi2|k_negcount_seg_xg|k_negcount_seg_y" -s 0 -c 40 \
    -o /tmp/s10_c3 python scripts/profile_solve.py C3 1 > $O/s10.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/s10_c3.ncu-rep $O/s10_c3.json C3 > /dev/null 2>&1; echo "sum rc=$?"
ncu -i /tmp/s10_c3.ncu-rep --page details --csv -k regex:"k_rqi2" > $O/s10_rqi2_details.csv 2>&1
