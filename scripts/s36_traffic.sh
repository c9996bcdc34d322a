#!/bin/bash
# ncu --set full of the dominant kernel (k_negcount_seg*) on the configurations whose bench line still had
# "traffic": null (C4, C5b, C5a, C1); each only after the plain run of the same command exited 0
O=gpurun_out
MIX="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fp64.sum"
python -c "import __graft_entry__ as g; g.build()" > $O/s36_build.log 2>&1 || exit 1
for C in C1 C4 C5b C5a; do
  python scripts/profile_solve.py $C 1 > $O/s36_plain_$C.log 2>&1 || { echo "plain $C failed"; continue; }
  # skip the warm rounds' first launches: capture 6 launches from the 10th on (mid rounds of the root bisection)
  timeout 600 ncu --set full --metrics $MIX --clock-control none -k regex:"k_negcount" -s 10 -c 6 \
      -o /tmp/s36_$C python scripts/profile_solve.py $C 1 > $O/s36_ncu_$C.log 2>&1; echo "ncu $C rc=$?"
  python scripts/ncu_summary.py /tmp/s36_$C.ncu-rep $O/ncu_summary_${C}_r02f_negseg.json $C > /dev/null 2>&1; echo "sum $C rc=$?"
  cp $O/ncu_summary_${C}_r02f_negseg.json profiles/ 2>/dev/null
done
for C in C4 C5b C5a C1; do
  timeout 1200 python bench.py --workload $C --steps 3 --warmup 3 --no-cpu-baseline > $O/r02f_bench_$C.json 2> $O/s36_bench_$C.err; echo "bench $C rc=$?"
done
