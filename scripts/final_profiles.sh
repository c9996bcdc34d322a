#!/bin/bash
# ncu evidence for the C2 headline: launch list of one solve + --set full of the dominant kernels
O=gpurun_out
python scripts/profile_solve.py C2 2 > $O/plain_final.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_final.csv \
    python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "launch list rc=$?"
# second solve: root rounds 1-3 of the segmented x-NegCount, then the RQI kernels and the z write
ncu --set full --clock-control none --import-source on -k regex:"k_negcount_seg" -s 35 -c 3 \
    -o $O/prof_negcount_C2_final python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu negcount rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_twist_lane|k_twist_pick2|k_fixed_chunk|k_zwrite_chunk|k_root<" \
    -s 7 -c 7 -o $O/prof_rqi_C2_final python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu rqi rc=$?"
