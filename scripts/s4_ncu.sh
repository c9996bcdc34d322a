O=gpurun_out
export MRRR_SEGK=16
python scripts/profile_solve.py C2 2 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_negcount_seg" -s 50 -c 1 \
    -o $O/s4b_negseg python scripts/profile_solve.py C2 2 > $O/s4b_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/s4b_negseg.ncu-rep --page details --csv > $O/s4b_details.csv 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.per_cycle_active --clock-control none -k regex:"k_negcount_seg" --csv --log-file $O/s4b_list.csv python scripts/profile_solve.py C2 1 > /dev/null 2>&1
unset MRRR_SEGK
ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.per_cycle_active --clock-control none -k regex:"k_negcount_seg" --csv --log-file $O/s4a_list.csv python scripts/profile_solve.py C2 1 > /dev/null 2>&1
