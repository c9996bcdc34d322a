#!/bin/bash
# round-2 final evidence after the numerical support + z recompute window: bench lines of every configuration
# (C2 with cpu_baseline and e2e), single/double and early-stop lines, launch lists (C2, C3, C4), ncu --set full
# of the root x-NegCount rounds and of the singleton-RQI kernels with the executed FP64 instruction mix
O=gpurun_out
MIX="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fp64.sum"
python bench.py > $O/r02b_bench_C2.json 2> $O/r02b_bench_C2.err; echo "bench C2 rc=$?"
for w in C1 C3 C4 C5b C5a; do
  st=5; [ $w = C5a ] && st=3
  python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/r02b_bench_$w.json 2> $O/r02b_bench_$w.err; echo "$w rc=$?"
done
for w in C1 C2; do
  python bench.py --profile sd --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02b_bench_sd_$w.json 2> $O/r02b_bench_sd_$w.err; echo "sd $w rc=$?"
done
python bench.py --early-stop --no-cpu-baseline > $O/r02b_bench_es_C2.json 2> $O/r02b_bench_es_C2.err; echo "es C2 rc=$?"
for w in C2 C3 C4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02b_launches_$w.csv \
      python scripts/profile_solve.py $w 2 > /dev/null 2>&1; echo "launch list $w rc=$?"
done
ncu --set full --metrics $MIX --clock-control none --import-source on -k regex:"k_negcount_seg" -s 35 -c 3 \
    -o $O/r02b_prof_negcount_C2 python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu negcount rc=$?"
ncu --set full --metrics $MIX --clock-control none --import-source on -k regex:"k_twist_lane|k_twist_pick2|k_fixed_chunk|k_zrc|k_zwrite_chunk" \
    -s 8 -c 8 -o $O/r02b_prof_rqi_C2 python scripts/profile_solve.py C2 2 > /dev/null 2>&1; echo "ncu rqi rc=$?"
ls -la $O/r02b_*
