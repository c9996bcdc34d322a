#!/bin/bash
# round-2 evidence run: GPU tests, C2 bench, launch list, ncu --set full of the dominant kernels with the
# executed FP64 instruction mix (scripts/ncu_summary.py)
O=gpurun_out
MIX="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fp64.sum"
python -m pytest tests -q -m gpu > $O/r02_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02_pytest.log
python bench.py > $O/r02_bench_C2.json 2> $O/r02_bench_C2.err; echo "bench rc=$?"
python scripts/profile_solve.py C2 2 > $O/r02_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_C2.csv \
    python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "launch list rc=$?"
ncu --set full --metrics $MIX --clock-control none --import-source on -k regex:"k_negcount_seg" -s 35 -c 3 \
    -o $O/r02_prof_negcount_C2 python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu negcount rc=$?"
ncu --set full --metrics $MIX --clock-control none --import-source on -k regex:"k_twist_lane|k_twist_pick2|k_fixed_chunk|k_zwrite_chunk|k_root<" \
    -s 7 -c 7 -o $O/r02_prof_rqi_C2 python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu rqi rc=$?"
