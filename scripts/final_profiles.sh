#!/bin/bash
# ncu evidence for the C2 headline: launch list of one solve + --set full of the two dominant kernels
O=gpurun_out
python scripts/profile_solve.py C2 2 > $O/plain_final.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_final.csv \
    python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_negcount_tma" -s 11 -c 3 \
    -o $O/prof_negcount_C2_final python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu negcount rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_rqi2|k_zwrite|k_root" -s 3 -c 3 \
    -o $O/prof_rqi_C2_final python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu rqi rc=$?"
