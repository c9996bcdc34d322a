# round-end numbers after the deferred tails + the C4 launch list
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/s34_build.log 2>&1 || exit 1
bash scripts/final_bench.sh
python scripts/profile_solve.py C4 2 > $O/s34_plain_C4.log 2>&1; echo "plain C4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_launches_C4.csv \
    python scripts/profile_solve.py C4 2 > /dev/null 2>&1; echo "launch list C4 rc=$?"
