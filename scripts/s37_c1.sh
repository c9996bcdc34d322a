#!/bin/bash
# C1: ncu --set full of the unsegmented root rounds (k_root), then the C1 and default bench lines with the final bench.py
O=gpurun_out
MIX="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fp64.sum"
python -c "import __graft_entry__ as g; g.build()" > $O/s37_build.log 2>&1 || exit 1
python scripts/profile_solve.py C1 1 > $O/s37_plain_C1.log 2>&1 || exit 1
timeout 600 ncu --set full --metrics $MIX --clock-control none -k regex:'^k_root$' -s 2 -c 6 \
    -o /tmp/s37_C1 python scripts/profile_solve.py C1 1 > $O/s37_ncu_C1.log 2>&1; echo "ncu C1 rc=$?"
python scripts/ncu_summary.py /tmp/s37_C1.ncu-rep $O/ncu_summary_C1_r02f_root.json C1 > /dev/null 2>&1; echo "sum C1 rc=$?"
cp $O/ncu_summary_C1_r02f_root.json profiles/ 2>/dev/null
timeout 600 python bench.py --workload C1 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02f_bench_C1.json 2> $O/s37_bench_C1.err; echo "bench C1 rc=$?"
timeout 900 python bench.py > $O/r02f_bench_C2.json 2> $O/s37_bench_C2.err; echo "bench C2 rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/s37_smoke.log 2>&1; echo "smoke rc=$?"
